#!/bin/bash
# configs[0] graph as text files, then the reference-style harness (bench_cli,
# cli.py:162-241) over the 8-combo grid with both GPU pipelines: the device
# text parser reads the files, `gpu` = encode(EdgeList) per repeat.
# (GPU box helper; writes gpurun_out/harness_*.txt)
python - <<'PY'
from oracle import gen
from paper_2406_03726_b200 import textio
from paper_2406_03726_b200.graph import EdgeList, LabelVector
c = gen.host_config(0)
with open("/tmp/sbm10k_edges.txt", "w") as f:
    textio.write_edge_list(EdgeList(c["n"], c["rows"], c["cols"], c["weights"]), f)
with open("/tmp/sbm10k_labels.txt", "w") as f:
    textio.write_labels(LabelVector(c["labels"], c["k"]), f)
PY
python -m paper_2406_03726_b200.bench_cli bench --edges /tmp/sbm10k_edges.txt --labels /tmp/sbm10k_labels.txt \
    --grid --pipeline both --repeats 5 --format table > gpurun_out/harness_table.txt 2> gpurun_out/harness_err.txt
echo "rc=$?"
