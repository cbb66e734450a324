"""Dense-state helpers for the TEBD tests (test infrastructure): restate the
reference's test helpers (tests/helpers.hpp mps_to_dense, apply_two_site,
schmidt_values) in numpy.  Dense index: site j is axis j of a Fortran-ordered
(d,)*n tensor (site 0 fastest)."""
from __future__ import annotations

import numpy as np


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def mps_to_dense(gammas, lambdas, charges):
    """psi(m_0..m_{n-1}) = lam_0 G_0[m_0] lam_1 G_1[m_1] ... lam_n with each
    bond space = [even sector; odd sector]."""
    d = len(charges)
    n = len(gammas)
    lam = [[_np(x) for x in pair] for pair in lambdas]
    dims = [(len(l[0]), len(l[1])) for l in lam]
    cplx = any(np.iscomplexobj(_np(x)) for site in gammas for pair in site for x in pair)

    def full_gamma(j, m):
        r0, r1 = dims[j]
        c0, c1 = dims[j + 1]
        g = np.zeros((r0 + r1, c0 + c1), dtype=np.complex128 if cplx else np.float64)
        for a in (0, 1):
            b = _np(gammas[j][m][a])
            ro = 0 if a == 0 else r0
            co = 0 if (a ^ charges[m]) == 0 else c0
            if b.size:
                g[ro:ro + b.shape[0], co:co + b.shape[1]] = b
        return g

    def full_lam(b):
        return np.concatenate([lam[b][0], lam[b][1]])

    # state as (d^j, bond_j) matrix built left to right
    cur = full_lam(0)[None, :]  # 1 x dim0
    for j in range(n):
        blocks = [cur @ full_gamma(j, m) * full_lam(j + 1)[None, :] for m in range(d)]
        # new row index = old_row + d^j * m  (site j is the slower digit here)
        cur = np.concatenate(blocks, axis=0)
    assert cur.shape[1] == 1
    return cur[:, 0]


def apply_two_site(v, gate_block, b, n, d):
    t = v.reshape((d,) * n, order="F")
    g = gate_block.reshape(d, d, d, d)  # [m1', m2', m1, m2]
    t = np.moveaxis(t, (b, b + 1), (0, 1))
    t = np.einsum("abcd,cd...->ab...", g, t)
    t = np.moveaxis(t, (0, 1), (b, b + 1))
    return t.reshape(-1, order="F")


def schmidt_values(v, cut, n, d):
    return np.linalg.svd(v.reshape(d ** cut, d ** (n - cut), order="F"), compute_uv=False)


def sorted_lambdas(lam_pair):
    return np.sort(np.concatenate([_np(lam_pair[0]), _np(lam_pair[1])]))[::-1]
