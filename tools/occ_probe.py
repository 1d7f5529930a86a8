import numpy as np, torch
import paper_2406_03726_b200 as G
from paper_2406_03726_b200 import synth
for n,k in ((10000,3),(3001,5)):
    rng=np.random.default_rng(0)
    r=rng.integers(0,n,50000); c=rng.integers(0,n,50000)
    e=G.EdgeList(n,r,c,np.ones(r.size),False)
    try:
        z=G.encode(e,G.LabelVector(rng.integers(0,k,n),k),G.EmbedOptions(True,True,True))
        print("ok",n,k)
    except Exception as ex: print("ERR",n,k,ex)
