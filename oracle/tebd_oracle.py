"""TEST INFRASTRUCTURE ONLY -- CPU restatement of rlftn's two-site bond update
(mps.cpp:62-108 random_product_state, mps.cpp:111-323 apply_gate) in numpy,
factorizing through the oracle's block_factorize restatement
(oracle/rsvd_oracle.cpp, blocks.cpp:38-118).  Only tests/ import it; the
product path (paper_1710_01463_b200/tebd.py) never does.

Parity pinned by: the reference's own MPS tests restated (tests/test_tebd_*),
gauge-invariant comparisons (Schmidt values, discarded weights, the truncated
two-site wavefunction) since singular-vector signs are a gauge freedom.
"""
from __future__ import annotations

import numpy as np

from . import oracle

LAMBDA_FLOOR = 1e-12
LAMBDA_TRIM = 1e-11


def _uniform(words):
    return ((words >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * (1.0 / 9007199254740992.0)


def random_product_state(charges, length, seed):
    """mps.cpp:62-108 -> (gammas[j][m][a], lambdas[b][s]) numpy."""
    d = len(charges)
    key = oracle.derive_seed(seed, 1)  # seed_tag::initial_state
    words = oracle.rng_words(key, 2 * length + 4)
    u = _uniform(words)
    ui = iter(u)

    def draw(n):
        return min(n - 1, int(next(ui) * float(n)))

    basis = [0] * length
    partial = 0
    for j in range(length - 1):
        basis[j] = draw(d)
        partial ^= charges[basis[j]]
    closing = [m for m in range(d) if charges[m] == partial]
    basis[length - 1] = closing[draw(len(closing))]
    cum = [0] * (length + 1)
    for j in range(length):
        cum[j + 1] = cum[j] ^ charges[basis[j]]
    lambdas = []
    for b in range(length + 1):
        pair = [np.zeros(0), np.zeros(0)]
        pair[cum[b]] = np.ones(1)
        lambdas.append(pair)
    gammas = []
    for j in range(length):
        site = []
        for m in range(d):
            pair = []
            for a in (0, 1):
                rows = 1 if a == cum[j] else 0
                cols = 1 if (a ^ charges[m]) == cum[j + 1] else 0
                pair.append(np.zeros((rows, cols)))
            site.append(pair)
        site[basis[j]][cum[j]][0, 0] = 1.0
        gammas.append(site)
    return gammas, lambdas


def apply_gate(gammas, lambdas, charges, bond, gate_block, gate_terms, form, chi, kind="tsvd",
               power=4, seed=0, oversample=0, min_dim=32, maximal=False, slack=-1):
    """mps.cpp:111-323.  gate_terms: [(left, right, charge)] for form "product".
    Updates gammas/lambdas in place; returns (discarded_weight, mid_rank, thetap)."""
    d = len(charges)
    p = charges
    lam_l, lam_m, lam_r = lambdas[bond], lambdas[bond + 1], lambdas[bond + 2]
    g1, g2 = gammas[bond], gammas[bond + 1]
    nl = [len(lam_l[0]), len(lam_l[1])]
    nm = [len(lam_m[0]), len(lam_m[1])]
    nr = [len(lam_r[0]), len(lam_r[1])]
    alm = [[lam_l[a][:, None] * g1[m][a] * lam_m[a ^ p[m]][None, :] for a in (0, 1)]
           for m in range(d)]
    br = [[g2[m][a] * lam_r[a ^ p[m]][None, :] for a in (0, 1)] for m in range(d)]
    row_off = [[0] * d, [0] * d]
    col_off = [[0] * d, [0] * d]
    rows, cols = [0, 0], [0, 0]
    for s in (0, 1):
        for m in range(d):
            row_off[s][m] = rows[s]
            rows[s] += nl[s ^ p[m]]
            col_off[s][m] = cols[s]
            cols[s] += nr[s ^ p[m]]
    thetap = [None, None]
    qfac = [None, None]
    lifted = False
    if form == "block":
        theta = []
        for s in (0, 1):
            if nm[s] == 0:
                theta.append(np.zeros((rows[s], cols[s])))
                continue
            astack = np.zeros((rows[s], nm[s]))
            bstack = np.zeros((nm[s], cols[s]))
            for m in range(d):
                astack[row_off[s][m]:row_off[s][m] + nl[s ^ p[m]], :] = alm[m][s ^ p[m]]
                bstack[:, col_off[s][m]:col_off[s][m] + nr[s ^ p[m]]] = br[m][s]
            theta.append(astack @ bstack)
        pairs = [[], []]
        for m1 in range(d):
            for m2 in range(d):
                pairs[p[m1] ^ p[m2]].append((m1, m2))
        gt = []
        for q in (0, 1):
            n = len(pairs[q])
            g = np.zeros((n, n))
            for i in range(n):
                for j in range(n):
                    g[i, j] = gate_block[pairs[q][j][0] * d + pairs[q][j][1],
                                         pairs[q][i][0] * d + pairs[q][i][1]]
            gt.append(g)
        thetap = [np.zeros((rows[sp], cols[sp])) for sp in (0, 1)]
        for a in (0, 1):
            for c in (0, 1):
                q = a ^ c
                n = len(pairs[q])
                blk = nl[a] * nr[c]
                if blk == 0 or n == 0:
                    continue
                tin = np.zeros((blk, n))
                for i, (m1, m2) in enumerate(pairs[q]):
                    s = a ^ p[m1]
                    sub = theta[s][row_off[s][m1]:row_off[s][m1] + nl[a],
                                   col_off[s][m2]:col_off[s][m2] + nr[c]]
                    tin[:, i] = sub.reshape(-1, order="F")
                tout = tin @ gt[q]
                for i, (m1, m2) in enumerate(pairs[q]):
                    sp = a ^ p[m1]
                    thetap[sp][row_off[sp][m1]:row_off[sp][m1] + nl[a],
                               col_off[sp][m2]:col_off[sp][m2] + nr[c]] = \
                        tout[:, i].reshape(nl[a], nr[c], order="F")
    else:
        for sp in (0, 1):
            koff, fused = [], 0
            for (_, _, ch) in gate_terms:
                koff.append(fused)
                fused += nm[sp ^ ch]
            x = np.zeros((rows[sp], fused))
            y = np.zeros((fused, cols[sp]))
            for k, (left, right, ch) in enumerate(gate_terms):
                w = nm[sp ^ ch]
                if w == 0:
                    continue
                for m1p in range(d):
                    a = sp ^ p[m1p]
                    if nl[a] == 0:
                        continue
                    for m1 in range(d):
                        if left[m1p, m1] != 0.0:
                            x[row_off[sp][m1p]:row_off[sp][m1p] + nl[a], koff[k]:koff[k] + w] += \
                                left[m1p, m1] * alm[m1][a]
                for m2p in range(d):
                    c = sp ^ p[m2p]
                    if nr[c] == 0:
                        continue
                    for m2 in range(d):
                        if right[m2p, m2] != 0.0:
                            y[koff[k]:koff[k] + w, col_off[sp][m2p]:col_off[sp][m2p] + nr[c]] += \
                                right[m2p, m2] * br[m2][sp ^ ch]
            if rows[sp] == 0 or fused == 0:
                qfac[sp] = np.zeros((rows[sp], 0))
                thetap[sp] = np.zeros((0, cols[sp]))
            else:
                qf, r = np.linalg.qr(x, mode="reduced")
                qfac[sp] = qf
                thetap[sp] = r @ y
        lifted = True
    total_sq = float(sum(np.sum(t * t) for t in thetap))
    if not total_sq > 0.0:
        raise RuntimeError("apply_gate: evolved wavefunction vanished")
    facs, _, _ = oracle.block_factorize(thetap, [0, 1], chi, maximal=maximal, slack=slack,
                                        kind=kind, oversample=oversample, power=power, seed=seed,
                                        min_dim=min_dim)
    facs = [list(f) for f in facs]  # [U, S, Vt, dw]
    kept_sq = float(sum(np.sum(f[1] ** 2) for f in facs))
    if kept_sq > 0.0:
        cut = LAMBDA_TRIM * np.sqrt(kept_sq)
        trimmed = False
        for f in facs:
            r = len(f[1])
            while r > 0 and f[1][r - 1] < cut:
                r -= 1
            if r == len(f[1]):
                continue
            f[0], f[1], f[2] = f[0][:, :r], f[1][:r], f[2][:r, :]
            trimmed = True
        if trimmed:
            kept_sq = float(sum(np.sum(f[1] ** 2) for f in facs))
    if not kept_sq > 0.0:
        raise RuntimeError("apply_gate: truncation removed the whole state")
    if lifted:
        for sp in (0, 1):
            facs[sp][0] = qfac[sp] @ facs[sp][0]
    inv = 1.0 / np.sqrt(kept_sq)
    for s in (0, 1):
        lam_m[s] = facs[s][1] * inv
    linv = [1.0 / np.maximum(lam_l[a], LAMBDA_FLOOR) for a in (0, 1)]
    rinv = [1.0 / np.maximum(lam_r[a], LAMBDA_FLOOR) for a in (0, 1)]
    for m in range(d):
        for a in (0, 1):
            s = a ^ p[m]
            g1[m][a] = linv[a][:, None] * facs[s][0][row_off[s][m]:row_off[s][m] + nl[a], :]
            g2[m][a] = (facs[a][2][:, col_off[a][m]:col_off[a][m] + nr[a ^ p[m]]] *
                        rinv[a ^ p[m]][None, :])
    return max(0.0, 1.0 - kept_sq / total_sq), len(lam_m[0]) + len(lam_m[1]), thetap


def canonicalize(gammas, lambdas, charges):
    """mps.cpp:326-350: identity gates right-to-left, left-to-right, then the
    even layer, exact factorization capped at d * max bond dimension."""
    d = len(charges)
    n = len(gammas)
    ident = np.eye(d * d)
    cap = d * max(len(l[0]) + len(l[1]) for l in lambdas)
    order = list(range(n - 2, -1, -1)) + list(range(n - 1)) + list(range(0, n - 1, 2))
    for b in order:
        apply_gate(gammas, lambdas, charges, b, ident, None, "block", cap, maximal=True)
