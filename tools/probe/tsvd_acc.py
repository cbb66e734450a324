import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1710_01463_b200 import tsvd, rsvd, RsvdParams
a = np.load("tests/golden/theta_rankdef_24x21.npy")
sv = np.linalg.svd(a, compute_uv=False)
for M in (a, a.T.copy()):
    f = tsvd(M, 200)
    sg = np.asarray(f.sigma)
    k = min(len(sg), 12)
    print(os.environ.get("TAG", ""), M.shape, "abs err", np.max(np.abs(sg[:k] - sv[:k])), "rank", len(sg))
f = rsvd(a, RsvdParams(15, 21, 0, 5))
print("rsvd q=0 l=21:", np.max(np.abs(np.asarray(f.sigma)[:12] - sv[:12])))
f = rsvd(a, RsvdParams(15, 21, 2, 5))
print("rsvd q=2 l=21:", np.max(np.abs(np.asarray(f.sigma)[:12] - sv[:12])))
