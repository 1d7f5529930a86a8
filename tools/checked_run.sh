# Rebuild libgee.so with device bounds assertions (make CHECKED=1), run the
# sanitize case and the stream / parity GPU tests under it, restore the normal build.
set -e
make -s -C paper_2406_03726_b200/csrc clean
make -s -j16 -C paper_2406_03726_b200/csrc CHECKED=1 > /dev/null
python tools/sanitize_case.py
python -m pytest tests/test_gpu_stream.py tests/test_gpu_gen.py tests/test_formats.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -q -x -k "fuzz or configs or fixture" 2>&1 | tail -2
make -s -C paper_2406_03726_b200/csrc clean
make -s -j16 -C paper_2406_03726_b200/csrc > /dev/null
