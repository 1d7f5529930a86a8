"""Debug helper: re-run one golden fixture case on the GPU and report where it differs."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from _golden import COMBOS, load, ztag
import paper_2406_03726_b200 as G
from oracle import oracle as O

name = sys.argv[1]
case = next(c for c in load() if c["name"] == name)
n, k, directed = case["n"], case["k"], case["directed"]
print("n", n, "k", k, "directed", directed, "m", case["rows"].size, "w uniq", np.unique(case["w"])[:8])
edges = G.EdgeList(n, case["rows"], case["cols"], case["w"], directed)
lab = G.LabelVector(case["labels"], k)
for lap, diag, corr in COMBOS:
    tag = ztag(lap, diag, corr)
    if tag + "_error" in case:
        continue
    opts = G.EmbedOptions(bool(lap), bool(diag), bool(corr))
    for nm, adj in (("edges", edges), ("csr", edges.to_csr())):
        z = G.encode(adj, lab, opts)
        d = np.abs(z - case[tag])
        if d.max() > 1e-12:
            r, c = np.unravel_index(np.argmax(d), d.shape)
            print(tag, nm, "max", d.max(), "at", r, c, "got", z[r], "ref", case[tag][r])
            ip, cc, vv = edges.to_csr().to_numpy()
            print("  row", r, "cols", cc[ip[r]:ip[r+1]], "vals", vv[ip[r]:ip[r+1]], "labels of cols", case["labels"][cc[ip[r]:ip[r+1]]])
            print("  ref row ptr", case["csr_indptr"][r:r+2], "ours", ip[r:r+2], "nnz", ip[-1], case["csr_indptr"][-1])
