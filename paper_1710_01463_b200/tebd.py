"""TEBD two-site bond update on the GPU: theta assembly, block factorization,
gauge update.

Mirrors rlftn's `apply_gate` (mps.cpp:111-323) on a Z2-symmetric MPS in the
Gamma/lambda gauge (mps.hpp:15-56), with every tensor resident on the device:

  * weighted site blocks alm = lam_l G1 lam_m, br = G2 lam_r (mps.cpp:130-137);
  * block form: theta_s = A_s B_s per middle sector, then the gate as one dense
    GEMM per pair charge on the scattered (a, c) blocks (mps.cpp:157-222);
    product form: the gate's Kronecker terms on the two halves, a per-sector
    QR of the left half and the factorization on the small core R Y
    (mps.cpp:223-266);
  * block_factorize over the two middle sectors (blocks.py, the engine),
    Schmidt trim at 1e-11 sqrt(kept), renormalisation and the inverse-lambda
    gauge update with the 1e-12 floor (mps.cpp:268-321).

`apply_gate_layer` updates a set of disjoint bonds (one TEBD layer,
mps.cpp:448-457) with ONE batched factorization: the sector blocks of all
bonds are grouped by shape into shared engine calls (blocks.block_factorize_many),
which is where the GPU wins over the reference's bond-by-bond loop.

The GEMMs of the assembly are plain cuBLAS calls through torch (library GEMMs
on chi-sized blocks) and the product-form QR is cuSOLVER's; the factorization
is the engine's.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from ._lib import InvalidArgument
from .blocks import (BlockDiagMatrix, BlockMethod, SectorRankRequest, block_factorize,
                     block_factorize_many)
from .models import GateForm, SiteStructure, TwoSiteGate
from .rng import CounterRng, derive_seed, seed_tag

LAMBDA_FLOOR = 1e-12  # mps.cpp:22
LAMBDA_TRIM = 1e-11   # mps.cpp:23


def _torch():
    import torch

    return torch


@dataclass
class GateStats:
    discarded_weight: float = 0.0
    factorize_seconds: float = 0.0
    mid_rank: int = 0


class SymmetricMPS:
    """mps.hpp:34-56: gammas[j][m][a] is a (len lam_j[a]) x (len lam_{j+1}[a ^ p(m)])
    device matrix, lambdas[b] = [even values, odd values]."""

    def __init__(self, site: SiteStructure, gammas, lambdas):
        self.site = site
        self.gammas = gammas
        self.lambdas = lambdas

    def length(self) -> int:
        return len(self.gammas)

    def bond_dimension(self, b: int) -> int:
        return int(self.lambdas[b][0].numel() + self.lambdas[b][1].numel())

    def max_bond_dimension(self) -> int:
        return max(self.bond_dimension(b) for b in range(self.length() + 1))

    def validate(self) -> None:
        """mps.cpp:39-60 (same checks and messages, as ValueError)."""
        n = self.length()
        if n < 1:
            raise ValueError("mps: no sites")
        if len(self.lambdas) != n + 1:
            raise ValueError("mps: need one bond more than sites")
        d = self.site.dim
        if d < 2 or len(self.site.charges) != d:
            raise ValueError("mps: invalid site structure")
        lz = self.lambdas
        if (lz[0][0].numel() != 1 or lz[0][1].numel() != 0 or lz[n][0].numel() != 1 or
                lz[n][1].numel() != 0):
            raise ValueError("mps: boundary bonds must be trivial even sectors")
        for j in range(n):
            if len(self.gammas[j]) != d:
                raise ValueError("mps: physical dimension mismatch")
            for m in range(d):
                for a in (0, 1):
                    b = self.gammas[j][m][a]
                    if (b.shape[0] != lz[j][a].numel() or
                            b.shape[1] != lz[j + 1][a ^ self.site.charges[m]].numel()):
                        raise ValueError("mps: block shape breaks the parity fusion rule")

    def to_numpy(self):
        """(gammas, lambdas) as numpy arrays (tests, oracle comparison)."""
        g = [[[x.cpu().numpy() for x in pair] for pair in site] for site in self.gammas]
        lam = [[x.cpu().numpy() for x in pair] for pair in self.lambdas]
        return g, lam


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


def _floored_inverse(lam):
    torch = _torch()
    return 1.0 / torch.clamp(lam, min=LAMBDA_FLOOR)


class _BondPlan:
    """Everything the update of one bond needs between its assembly and its
    gauge update (sector offsets, the assembled theta', QR factors)."""


def _assemble(psi: SymmetricMPS, bond: int, gate: TwoSiteGate) -> _BondPlan:
    """mps.cpp:111-266: the two-site matrix theta' as a 2-sector block matrix."""
    torch = _torch()
    n_sites = psi.length()
    if bond < 0 or bond + 1 >= n_sites:
        raise InvalidArgument("apply_gate: bond out of range")
    d = psi.site.dim
    p = psi.site.charges
    if gate.block is None or gate.block.shape != (d * d, d * d):
        raise InvalidArgument("apply_gate: gate does not match the physical dimension")
    lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
    g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
    dev = lam_l[0].device
    # theta carries the Gammas' scalar type (real or complex MPS); gates are real.
    f64 = dict(dtype=g1[0][0].dtype, device=dev)
    nl = [lam_l[0].numel(), lam_l[1].numel()]
    nm = [lam_m[0].numel(), lam_m[1].numel()]
    nr = [lam_r[0].numel(), lam_r[1].numel()]
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
    plan = _BondPlan()
    plan.bond, plan.nl, plan.nm, plan.nr = bond, nl, nm, nr
    plan.row_off, plan.col_off, plan.rows, plan.cols = row_off, col_off, rows, cols
    plan.lifted = False
    plan.qfac = [None, None]
    thetap = [None, None]
    if gate.form == GateForm.block:
        theta = []
        for s in (0, 1):
            if nm[s] == 0:
                theta.append(torch.zeros(rows[s], cols[s], **f64))
                continue
            astack = torch.cat([alm[m][s ^ p[m]] for m in range(d)], dim=0)
            bstack = torch.cat([br[m][s] for m in range(d)], dim=1)
            theta.append(astack @ bstack)
        pairs = [[], []]
        for m1 in range(d):
            for m2 in range(d):
                pairs[p[m1] ^ p[m2]].append((m1, m2))
        # theta' columns = theta columns * gt, gt(i, j) = gate(pair_j, pair_i);
        # built once per (gate, scalar type, device) and cached on the gate.
        cache = gate.__dict__.setdefault("_device_blocks", {})
        ckey = (f64["dtype"], str(dev), tuple(p))
        gt = cache.get(ckey)
        if gt is None:
            gblock = torch.as_tensor(gate.block, **f64)
            gt = []
            for q in (0, 1):
                idx = torch.tensor([m1 * d + m2 for (m1, m2) in pairs[q]], device=dev,
                                   dtype=torch.long)
                gt.append(gblock[idx][:, idx].t().contiguous() if len(pairs[q]) else None)
            cache[ckey] = gt
        thetap = [torch.zeros(rows[sp], cols[sp], **f64) for sp in (0, 1)]
        for a in (0, 1):
            for c in (0, 1):
                q = a ^ c
                npair = len(pairs[q])
                blk = nl[a] * nr[c]
                if blk == 0 or npair == 0:
                    continue
                # the (m1, m2) blocks of this (a, c) stacked, mixed by the gate in
                # one product: block'_j = sum_i gt(i, j) block_i
                tin = torch.stack([
                    theta[a ^ p[m1]][row_off[a ^ p[m1]][m1]:row_off[a ^ p[m1]][m1] + nl[a],
                                     col_off[a ^ p[m1]][m2]:col_off[a ^ p[m1]][m2] + nr[c]]
                    for (m1, m2) in pairs[q]])
                tout = (gt[q].t() @ tin.reshape(npair, blk)).reshape(npair, nl[a], nr[c])
                for i, (m1, m2) in enumerate(pairs[q]):
                    sp = a ^ p[m1]
                    thetap[sp][row_off[sp][m1]:row_off[sp][m1] + nl[a],
                               col_off[sp][m2]:col_off[sp][m2] + nr[c]] = tout[i]
    else:
        if not gate.terms:
            raise InvalidArgument("apply_gate: product-form gate has no terms")
        nk = len(gate.terms)
        for sp in (0, 1):
            koff = []
            fused = 0
            for t in gate.terms:
                koff.append(fused)
                fused += nm[sp ^ t.charge]
            x = torch.zeros(rows[sp], fused, **f64)
            y = torch.zeros(fused, cols[sp], **f64)
            for k in range(nk):
                t = gate.terms[k]
                w = nm[sp ^ t.charge]
                if w == 0:
                    continue
                for m1p in range(d):
                    a = sp ^ p[m1p]
                    if nl[a] == 0:
                        continue
                    xb = x[row_off[sp][m1p]:row_off[sp][m1p] + nl[a], koff[k]:koff[k] + w]
                    for m1 in range(d):
                        if t.left[m1p, m1] != 0.0:
                            xb += float(t.left[m1p, m1]) * alm[m1][a]
                for m2p in range(d):
                    c = sp ^ p[m2p]
                    if nr[c] == 0:
                        continue
                    yb = y[koff[k]:koff[k] + w, col_off[sp][m2p]:col_off[sp][m2p] + nr[c]]
                    for m2 in range(d):
                        if t.right[m2p, m2] != 0.0:
                            yb += float(t.right[m2p, m2]) * br[m2][sp ^ t.charge]
            if rows[sp] == 0 or fused == 0:
                plan.qfac[sp] = torch.zeros(rows[sp], 0, **f64)
                thetap[sp] = torch.zeros(0, cols[sp], **f64)
            else:
                qf, r = torch.linalg.qr(x, mode="reduced")
                plan.qfac[sp] = qf
                thetap[sp] = r @ y
        plan.lifted = True
    plan.thetap = thetap
    # kept on the device: the callers read all bonds' norms in one transfer
    plan.total_sq_t = sum((tp.abs() ** 2).sum() if tp.is_complex() else (tp * tp).sum()
                          for tp in thetap)
    return plan


def _read_norms(plans) -> None:
    """One device -> host transfer for every plan's ||theta'||^2 (mps.cpp:268)."""
    torch = _torch()
    vals = torch.stack([torch.as_tensor(p.total_sq_t, dtype=torch.float64,
                                        device=p.thetap[0].device).reshape(())
                        for p in plans]).cpu().tolist()
    for p, v in zip(plans, vals):
        p.total_sq = float(v)
        if not (p.total_sq > 0.0):
            raise RuntimeError("apply_gate: evolved wavefunction vanished")


def _finish(psi: SymmetricMPS, plan: _BondPlan, f, seconds: float) -> GateStats:
    """mps.cpp:276-321: trim, renormalise, lift, gauge update."""
    torch = _torch()
    factors = f.factors
    # host copies of the kept values (blocks._select), no per-sector transfer
    sh = [getattr(x, "sigma_host", None) for x in factors]
    sh = [v if v is not None else (x.sigma.cpu().numpy() if hasattr(x.sigma, "cpu")
                                   else np.asarray(x.sigma)) for v, x in zip(sh, factors)]
    kept_sq = float(sum(float(np.dot(v, v)) for v in sh))
    if kept_sq > 0.0:
        cut = LAMBDA_TRIM * np.sqrt(kept_sq)
        trimmed = False
        for i, fac in enumerate(factors):
            sv = sh[i]
            r = len(sv)
            while r > 0 and sv[r - 1] < cut:
                r -= 1
            if r == len(sv):
                continue
            fac.left = fac.left[:, :r]
            fac.sigma = fac.sigma[:r]
            fac.right_adj = fac.right_adj[:r, :]
            sh[i] = sv[:r]
            fac.sigma_host = sh[i]
            trimmed = True
        if trimmed:
            kept_sq = float(sum(float(np.dot(v, v)) for v in sh))
    if not (kept_sq > 0.0):
        raise RuntimeError("apply_gate: truncation removed the whole state")
    if plan.lifted:
        for sp in (0, 1):
            factors[sp].left = plan.qfac[sp] @ factors[sp].left
    bond = plan.bond
    d = psi.site.dim
    p = psi.site.charges
    lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
    inv_norm = 1.0 / np.sqrt(kept_sq)
    for s in (0, 1):
        lam_m[s] = factors[s].sigma * inv_norm
    linv = [_floored_inverse(lam_l[0]), _floored_inverse(lam_l[1])]
    rinv = [_floored_inverse(lam_r[0]), _floored_inverse(lam_r[1])]
    g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
    nl, nr = plan.nl, plan.nr
    for m in range(d):
        for a in (0, 1):
            s = a ^ p[m]
            lrows = factors[s].left[plan.row_off[s][m]:plan.row_off[s][m] + nl[a], :]
            g1[m][a] = linv[a][:, None] * lrows
            rcols = factors[a].right_adj[:, plan.col_off[a][m]:plan.col_off[a][m] + nr[a ^ p[m]]]
            g2[m][a] = rcols * rinv[a ^ p[m]][None, :]
    out = GateStats()
    out.discarded_weight = max(0.0, 1.0 - kept_sq / plan.total_sq)
    out.factorize_seconds = seconds
    out.mid_rank = int(lam_m[0].numel() + lam_m[1].numel())
    return out


def apply_gate(psi: SymmetricMPS, bond: int, gate: TwoSiteGate, chi: int, method: BlockMethod,
               request: Optional[SectorRankRequest] = None, handle=None) -> GateStats:
    """rlftn::apply_gate (mps.cpp:111-323) on device-resident tensors."""
    if chi < 1:
        raise InvalidArgument("apply_gate: chi must be >= 1")
    request = request or SectorRankRequest()
    plan = _assemble(psi, bond, gate)
    _read_norms([plan])
    torch = _torch()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = block_factorize(BlockDiagMatrix([0, 1], plan.thetap), chi, request, method, handle)
    torch.cuda.synchronize()
    return _finish(psi, plan, f, time.perf_counter() - t0)


def apply_gate_layer(psi: SymmetricMPS, bonds: Sequence[int], gates: Sequence[TwoSiteGate],
                     chi: int, method: BlockMethod, request: Optional[SectorRankRequest] = None,
                     handle=None) -> List[GateStats]:
    """One TEBD layer: gates on disjoint bonds (mps.cpp:448-457), all theta'
    assembled first, then ONE batched block factorization for all bonds
    (equal-shape sector blocks of different bonds share engine calls), then
    the per-bond gauge updates.  Same result as applying the gates one by
    one."""
    if chi < 1:
        raise InvalidArgument("apply_gate: chi must be >= 1")
    if len(bonds) != len(gates):
        raise InvalidArgument("apply_gate_layer: one gate per bond")
    used = set()
    for b in bonds:
        if b in used or b - 1 in used or b + 1 in used:
            raise InvalidArgument("apply_gate_layer: bonds must be disjoint")
        used.add(b)
    request = request or SectorRankRequest()
    plans = [_assemble(psi, b, g) for b, g in zip(bonds, gates)]
    _read_norms(plans)
    torch = _torch()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fs = block_factorize_many([BlockDiagMatrix([0, 1], pl.thetap) for pl in plans], chi, request,
                              method, handle)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return [_finish(psi, pl, f, dt / max(len(plans), 1)) for pl, f in zip(plans, fs)]


def canonicalize(psi: SymmetricMPS, handle=None) -> None:
    """rlftn::canonicalize (mps.cpp:326-350): identity gates right-to-left,
    left-to-right, then one even-bond layer, exact factorization with the cap
    d * max bond dimension (identity gates cannot raise a rank)."""
    from .blocks import RankPolicy

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
