"""Large sample widths l (real up to 1100, complex up to 1024) against the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle
from tests.helpers import matrix_with_spectrum, zmatrix_with_spectrum, rel_sigma_err
from paper_1710_01463_b200 import RsvdParams, rsvd, tsvd
oracle.set_threads(16)
for kind, m, n, ells in (("real", 1400, 1200, (700, 900, 1100)), ("complex", 1200, 1100, (432, 480, 512, 700, 1024))):
    mk = matrix_with_spectrum if kind == "real" else zmatrix_with_spectrum
    ref_fn = oracle.rsvd if kind == "real" else oracle.zrsvd
    a = mk(oracle, 77, m, n, np.exp(-np.arange(min(m, n)) / 200.0))
    for ell in ells:
        k = ell // 2
        try:
            t0 = time.time()
            f = rsvd(a, RsvdParams(k, ell, 1, 3))
            t1 = time.time()
            S = ref_fn(a, k, ell, 1, 3)[1]
            print(kind, ell, "ok", f.rank(), len(S), "sigma rel err %.2e" % rel_sigma_err(f.sigma, S), "%.2fs" % (t1 - t0), flush=True)
        except Exception as e:
            print(kind, ell, "ERR", e, flush=True)
