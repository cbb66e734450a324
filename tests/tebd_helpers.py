"""Dense-state helpers for the TEBD tests (test infrastructure): restate the
reference's test helpers (tests/helpers.hpp mps_to_dense, apply_two_site,
schmidt_values) in numpy, and the state preparation the bond-update tests
start from (mps.cpp random_product_state / canonicalize / lambda audits,
moved out of the product: only apply_gate / apply_gate_layer are on the
path).  Dense index: site j is axis j of a Fortran-ordered
(d,)*n tensor (site 0 fastest)."""
from __future__ import annotations

import numpy as np

from paper_1710_01463_b200._lib import InvalidArgument
from paper_1710_01463_b200.blocks import BlockMethod, RankPolicy, SectorRankRequest
from paper_1710_01463_b200.gates import GateForm, SiteStructure, TwoSiteGate
from paper_1710_01463_b200.rng import CounterRng, derive_seed, seed_tag
from paper_1710_01463_b200.tebd import SymmetricMPS, apply_gate, apply_gate_layer


def _torch():
    import torch

    return torch


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


def random_product_state(site: SiteStructure, length: int, seed: int,
                         device="cuda", dtype=None) -> SymmetricMPS:
    """mps.cpp:62-108: uniform basis states from
    CounterRng(derive_seed(seed, initial_state)), the last site closing the
    total parity to even.  ``dtype`` torch.complex128 gives the
    SymmetricMPS<Complex> instantiation (mps.cpp:551-555): complex Gammas (the
    bond updates then run the complex factorization), real lambdas."""
    torch = _torch()
    if length < 2:
        raise InvalidArgument("random_product_state: need at least two sites")
    d = site.dim
    if d < 2 or len(site.charges) != d:
        raise InvalidArgument("random_product_state: invalid site structure")
    rng = CounterRng(derive_seed(seed, seed_tag.initial_state))

    def draw(n):
        return min(n - 1, int(rng.uniform() * float(n)))

    basis = [0] * length
    partial = 0
    for j in range(length - 1):
        basis[j] = draw(d)
        partial ^= site.charges[basis[j]]
    closing = [m for m in range(d) if site.charges[m] == partial]
    if not closing:
        raise InvalidArgument("random_product_state: parity not closable")
    basis[length - 1] = closing[draw(len(closing))]
    cum = [0] * (length + 1)
    for j in range(length):
        cum[j + 1] = cum[j] ^ site.charges[basis[j]]
    f64 = dict(dtype=torch.float64, device=device)
    gdt = dict(dtype=dtype or torch.float64, device=device)
    lambdas = []
    for b in range(length + 1):
        pair = [torch.zeros(0, **f64), torch.zeros(0, **f64)]
        pair[cum[b]] = torch.ones(1, **f64)
        lambdas.append(pair)
    gammas = []
    for j in range(length):
        site_t = []
        for m in range(d):
            pair = []
            for a in (0, 1):
                rows = 1 if a == cum[j] else 0
                cols = 1 if (a ^ site.charges[m]) == cum[j + 1] else 0
                pair.append(torch.zeros(rows, cols, **gdt))
            site_t.append(pair)
        site_t[basis[j]][cum[j]][0, 0] = 1.0
        gammas.append(site_t)
    return SymmetricMPS(site, gammas, lambdas)


def canonicalize(psi: SymmetricMPS, handle=None) -> None:
    """rlftn::canonicalize (mps.cpp:326-350): identity gates right-to-left,
    left-to-right, then one even-bond layer, exact factorization with the cap
    d * max bond dimension (identity gates cannot raise a rank)."""
    psi.validate()
    n = psi.length()
    d = psi.site.dim
    ident = TwoSiteGate(GateForm.block, 0.0, np.eye(d * d), [])
    req = SectorRankRequest(RankPolicy.maximal, 0)
    exact = BlockMethod.deterministic()
    cap = d * psi.max_bond_dimension()
    for b in range(n - 2, -1, -1):
        apply_gate(psi, b, ident, cap, exact, req, handle)
    for b in range(n - 1):
        apply_gate(psi, b, ident, cap, exact, req, handle)
    layer = list(range(0, n - 1, 2))
    apply_gate_layer(psi, layer, [ident] * len(layer), cap, exact, req, handle)


def lambda_norm_error(psi: SymmetricMPS) -> float:
    """mps.cpp:352-358: max_b |sum lambda_b^2 - 1|."""
    return max(abs(float((l[0] * l[0]).sum() + (l[1] * l[1]).sum()) - 1.0) for l in psi.lambdas)
