#!/bin/bash
# configs[0] graph as text files, then the reference-style harness over the 8-combo grid
# with both GPU pipelines (GPU box helper; writes gpurun_out/harness_*.txt)
python - <<'PY'
from paper_2406_03726_b200 import synth, formats as F
from paper_2406_03726_b200.graph import EdgeList, LabelVector
c = synth.make_config(0)
with open("/tmp/sbm10k_edges.txt", "w") as f:
    F.write_edge_list(EdgeList(c["n"], c["rows"], c["cols"], c["weights"]), f)
with open("/tmp/sbm10k_labels.txt", "w") as f:
    F.write_labels(LabelVector(c["labels"], c["k"]), f)
PY
python -m paper_2406_03726_b200.bench_cli bench --edges /tmp/sbm10k_edges.txt --labels /tmp/sbm10k_labels.txt \
    --grid --pipeline both --repeats 3 --format table > gpurun_out/harness_table.txt 2> gpurun_out/harness_err.txt
echo "rc=$?"
