import numpy as np, sys
sys.path.insert(0, '.')
from paper_1710_01463_b200 import RsvdParams, rsvd, tsvd
g = np.load("tests/golden/zrsvd_small.npz")
for name in sorted({k.split("/")[0] for k in g.files}):
    a = g[f"{name}/a"]
    k, ell, q, seed = (int(x) for x in g[f"{name}/params"])
    for what in ("rsvd", "tsvd"):
        try:
            f = rsvd(a, RsvdParams(k, ell, q, seed)) if what == "rsvd" else tsvd(a, k)
            print(name, what, a.shape, "ok")
        except Exception as e:
            print(name, what, a.shape, k, ell, q, "ERR", e)
    ar = a.real.copy()
    try:
        rsvd(np.asfortranarray(np.vstack([ar, ar])[:a.shape[0]]), RsvdParams(k, ell, q, seed))
    except Exception as e:
        print("real", name, e)
