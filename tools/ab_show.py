"""Print step and top-kernel times of A/B bench lines: python tools/ab_show.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = [json.loads(x) for x in open(f) if x.startswith("{")][-1]
    except (IndexError, OSError):
        print(f, "missing")
        continue
    print(f"{f:36s} {d['ms_per_step']:8.3f} ms", " ".join(f"{k['kernel']}={k['ms_per_launch']:.3f}" for k in d["kernels"][:8]))
