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

Every arithmetic step runs on the engine's own kernels through the C ABI:
the lambda weighting, stacking, gate mixing, Kronecker sums, theta norms and
gauge update are table-driven launches covering the whole layer
(rsvd_combine_blocks / rsvd_block_sqnorms), the theta products, the
product-form core R y and the lift Q U are one grouped GEMM launch each
(rsvd_grouped_gemm), and the product-form QR is the engine's CholeskyQR2
(rsvd_qr_f64, batched per shape).  torch only allocates device memory.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument
from .blocks import (BlockDiagMatrix, BlockMethod, SectorRankRequest, block_factorize,
                     block_factorize_many)
from .gates import GateForm, SiteStructure, TwoSiteGate

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


def _floored_inverse(lam):
    torch = _torch()
    return 1.0 / torch.clamp(lam, min=LAMBDA_FLOOR)


class _BondPlan:
    """Everything the update of one bond needs between its assembly and its
    gauge update (sector offsets, the assembled theta', QR factors)."""


def _colmajor(rows: int, cols: int, like):
    """Uninitialised device matrix in column-major storage (the engine's
    layout; the table kernels write it row-fastest, i.e. coalesced)."""
    torch = _torch()
    return torch.empty((cols, rows), dtype=like.dtype, device=like.device).t()


class _Tables:
    """Host job tables of one launch of the engine's table-driven bond-update
    kernels (rsvd_combine_blocks / rsvd_grouped_gemm / rsvd_block_sqnorms)."""

    def __init__(self):
        self.jobs, self.terms, self.gemms = [], [], []
        self.keep = []  # tensors whose storage the tables point to

    @staticmethod
    def _view(t):
        return t.data_ptr(), t.stride(0), t.stride(1)

    def combine(self, dst, terms):
        """dst = sum_t coef * diag(row_scale) src diag(col_scale); terms =
        [(src, row_scale or None, col_scale or None, coef)]."""
        rows, cols = dst.shape
        if rows == 0 or cols == 0:
            return
        begin = len(self.terms)
        for src, rsc, csc, coef in terms:
            if coef == 0:
                continue
            sp, srs, scs = self._view(src)
            c = complex(coef)
            self.terms.append((sp, srs, scs, rsc.data_ptr() if rsc is not None else 0,
                               csc.data_ptr() if csc is not None else 0, c.real, c.imag))
            self.keep.append(src)
        dp, drs, dcs = self._view(dst)
        self.jobs.append((dp, drs, dcs, rows, cols, begin, len(self.terms) - begin))
        self.keep.append(dst)

    def gemm(self, c, a, b):
        if c.shape[0] == 0 or c.shape[1] == 0:
            return
        if a.shape[1] == 0:
            self.combine(c, [])
            return
        ap, ars, acs = self._view(a)
        bp, brs, bcs = self._view(b)
        cp, crs, ccs = self._view(c)
        self.gemms.append((ap, ars, acs, bp, brs, bcs, cp, crs, ccs, c.shape[0], c.shape[1],
                           a.shape[1]))
        self.keep += [a, b, c]

    def run_combine(self, h, cplx: bool):
        lib = _lib.load()
        if not self.jobs:
            return
        jobs = np.array(self.jobs, dtype=_lib.BLOCK_JOB)
        terms = np.array(self.terms, dtype=_lib.BLOCK_TERM) if self.terms else \
            np.zeros(1, dtype=_lib.BLOCK_TERM)
        _lib.raise_for(lib.rsvd_combine_blocks(h.raw, int(cplx), len(jobs), jobs.ctypes.data,
                                               len(self.terms), terms.ctypes.data), h.raw)
        self.jobs, self.terms = [], []

    def run_gemm(self, h, cplx: bool):
        lib = _lib.load()
        if not self.gemms:
            return
        g = np.array(self.gemms, dtype=_lib.GEMM_JOB)
        _lib.raise_for(lib.rsvd_grouped_gemm(h.raw, int(cplx), len(g), g.ctypes.data), h.raw)
        self.gemms = []


def _bond_sizes(psi: SymmetricMPS, bond: int, gate: TwoSiteGate) -> _BondPlan:
    """Validation and sector bookkeeping of apply_gate (mps.cpp:114-156)."""
    n_sites = psi.length()
    if bond < 0 or bond + 1 >= n_sites:
        raise InvalidArgument("apply_gate: bond out of range")
    d = psi.site.dim
    p = psi.site.charges
    if gate.block is None or gate.block.shape != (d * d, d * d):
        raise InvalidArgument("apply_gate: gate does not match the physical dimension")
    if gate.form != GateForm.block and not gate.terms:
        raise InvalidArgument("apply_gate: product-form gate has no terms")
    lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
    nl = [lam_l[0].numel(), lam_l[1].numel()]
    nm = [lam_m[0].numel(), lam_m[1].numel()]
    nr = [lam_r[0].numel(), lam_r[1].numel()]
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
    plan.bond, plan.gate, plan.nl, plan.nm, plan.nr = bond, gate, nl, nm, nr
    plan.row_off, plan.col_off, plan.rows, plan.cols = row_off, col_off, rows, cols
    plan.qfac = [None, None]
    plan.thetap = [None, None]
    return plan


def _assemble_layer(psi: SymmetricMPS, plans: List[_BondPlan], handle) -> None:
    """mps.cpp:111-268 for every bond of `plans`: theta' of each bond as a
    2-sector block matrix, in four engine launches for the whole layer --
    (1) the lambda-weighted site blocks written into the stacked operands
    (block form) or the Kronecker sums x, y (product form); (2) the grouped
    products theta_mu = Astack_mu Bstack_mu; (3) the gate mixing of the
    (m1, m2) blocks into theta'; (4) ||theta'||^2 per bond -- plus, for the
    product form, one batched CholeskyQR2 per shape (x = Q R) and the grouped
    core products R y.  No library GEMM or factorization is called."""
    torch = _torch()
    h = handle or _lib.default_handle()
    d = psi.site.dim
    p = psi.site.charges
    ref = psi.gammas[0][0][0]
    cplx = ref.is_complex()
    dev = ref.device
    st1, st2, st3 = _Tables(), _Tables(), _Tables()
    qr_groups = {}  # (rows, fused) -> [(plan, sp, x, y)]
    lifted_y = []   # (plan, sp, x, y) multiplied directly (no QR)
    for pl in plans:
        bond = pl.bond
        lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
        g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
        nl, nm, nr, rows, cols = pl.nl, pl.nm, pl.nr, pl.rows, pl.cols
        gate = pl.gate
        if gate.form == GateForm.block:
            pl.lifted = False
            theta = [None, None]
            for mu in (0, 1):
                if nm[mu] == 0:
                    continue
                A = _colmajor(rows[mu], nm[mu], ref)
                B = _colmajor(nm[mu], cols[mu], ref)
                for m in range(d):
                    a = mu ^ p[m]
                    st1.combine(A[pl.row_off[mu][m]:pl.row_off[mu][m] + nl[a]],
                                [(g1[m][a], lam_l[a], lam_m[mu], 1.0)])
                    c = mu ^ p[m]
                    st1.combine(B[:, pl.col_off[mu][m]:pl.col_off[mu][m] + nr[c]],
                                [(g2[m][mu], None, lam_r[c], 1.0)])
                theta[mu] = _colmajor(rows[mu], cols[mu], ref)
                st2.gemm(theta[mu], A, B)
            gb = gate.block
            thetap = [_colmajor(rows[sp], cols[sp], ref) for sp in (0, 1)]
            for sp in (0, 1):
                for m1 in range(d):
                    a = sp ^ p[m1]
                    for m2 in range(d):
                        c = sp ^ p[m2]
                        q = p[m1] ^ p[m2]
                        out = thetap[sp][pl.row_off[sp][m1]:pl.row_off[sp][m1] + nl[a],
                                         pl.col_off[sp][m2]:pl.col_off[sp][m2] + nr[c]]
                        terms = []
                        for i1 in range(d):
                            for i2 in range(d):
                                if p[i1] ^ p[i2] != q:
                                    continue
                                coef = float(gb[m1 * d + m2, i1 * d + i2])
                                mu = a ^ p[i1]
                                if coef == 0.0 or theta[mu] is None:
                                    continue
                                src = theta[mu][pl.row_off[mu][i1]:pl.row_off[mu][i1] + nl[a],
                                                pl.col_off[mu][i2]:pl.col_off[mu][i2] + nr[c]]
                                terms.append((src, None, None, coef))
                        st3.combine(out, terms)
            pl.thetap = thetap
        else:
            pl.lifted = True
            for sp in (0, 1):
                koff, fused = [], 0
                for t in gate.terms:
                    koff.append(fused)
                    fused += nm[sp ^ t.charge]
                x = _colmajor(rows[sp], fused, ref)
                y = _colmajor(fused, cols[sp], ref)
                for k, t in enumerate(gate.terms):
                    mu = sp ^ t.charge
                    w = nm[mu]
                    if w == 0:
                        continue
                    for m1p in range(d):
                        a = sp ^ p[m1p]
                        st1.combine(x[pl.row_off[sp][m1p]:pl.row_off[sp][m1p] + nl[a],
                                      koff[k]:koff[k] + w],
                                    [(g1[m1][a], lam_l[a], lam_m[mu], float(t.left[m1p, m1]))
                                     for m1 in range(d) if t.left[m1p, m1] != 0.0])
                    for m2p in range(d):
                        c = sp ^ p[m2p]
                        st1.combine(y[koff[k]:koff[k] + w,
                                      pl.col_off[sp][m2p]:pl.col_off[sp][m2p] + nr[c]],
                                    [(g2[m2][mu], None, lam_r[c], float(t.right[m2p, m2]))
                                     for m2 in range(d) if t.right[m2p, m2] != 0.0])
                if rows[sp] == 0 or fused == 0:  # mps.cpp:256-258
                    pl.qfac[sp] = torch.zeros(rows[sp], 0, dtype=ref.dtype, device=dev)
                    pl.thetap[sp] = torch.zeros(0, cols[sp], dtype=ref.dtype, device=dev)
                    continue
                if not cplx and rows[sp] > fused:
                    qr_groups.setdefault((rows[sp], fused), []).append((pl, sp, x, y))
                else:
                    # no reduction possible (or complex state): theta' = x y with
                    # qfac = I -- the same factorization, exactly, as Q (R y)
                    pl.qfac[sp] = None
                    pl.thetap[sp] = _colmajor(rows[sp], cols[sp], ref)
                    lifted_y.append((pl, sp, x, y))
    # (1) weighted site blocks / Kronecker sums
    with _lib.on_torch_stream(h):
        st1.run_combine(h, cplx)
        # product form: batched CholeskyQR2 per (rows, fused) shape, then R y
        for (m, n), members in qr_groups.items():
            nb = len(members)
            X = torch.empty((nb, n, m), dtype=ref.dtype, device=dev)
            Xv = X.transpose(1, 2)
            for i, (_, _, x, _) in enumerate(members):
                Xv[i].copy_(x)
            Qb = torch.empty((nb, n, m), dtype=ref.dtype, device=dev).transpose(1, 2)
            Rb = torch.empty((nb, n, n), dtype=ref.dtype, device=dev).transpose(1, 2)
            lib = _lib.load()
            _lib.raise_for(lib.rsvd_qr_f64(h.raw, nb, Xv.data_ptr(), m, n, m, m * n,
                                           Qb.data_ptr(), m, m * n, Rb.data_ptr(), n, n * n,
                                           _lib.PTR_DEVICE), h.raw)
            for i, (pl, sp, _, y) in enumerate(members):
                pl.qfac[sp] = Qb[i]
                pl.thetap[sp] = _colmajor(n, pl.cols[sp], ref)
                st2.gemm(pl.thetap[sp], Rb[i], y)
        for pl, sp, x, y in lifted_y:
            st2.gemm(pl.thetap[sp], x, y)
        # (2) theta_mu = Astack Bstack, R y, x y
        st2.run_gemm(h, cplx)
        # (3) gate mixing
        st3.run_combine(h, cplx)
        # (4) ||theta'||^2 per bond, one device -> host transfer for the layer
        blocks, begin = [], [0]
        for pl in plans:
            for tp in pl.thetap:
                if tp is not None and tp.numel():
                    dp_, rs_, cs_ = _Tables._view(tp)
                    blocks.append((dp_, rs_, cs_, tp.shape[0], tp.shape[1], 0, 0))
            begin.append(len(blocks))
        out = torch.empty(len(plans), dtype=torch.float64, device=dev)
        bt = np.array(blocks if blocks else [(0, 0, 0, 0, 0, 0, 0)], dtype=_lib.BLOCK_JOB)
        bg = np.array(begin, dtype=np.int64)
        lib = _lib.load()
        _lib.raise_for(lib.rsvd_block_sqnorms(h.raw, int(cplx), len(plans), bg.ctypes.data,
                                              bt.ctypes.data, out.data_ptr()), h.raw)
        vals = out.cpu().tolist()
    # keep every table operand alive until the stream has consumed it
    for pl, v in zip(plans, vals):
        pl.total_sq = float(v)
        pl._keep = (st1.keep, st2.keep, st3.keep)
        if not (pl.total_sq > 0.0):
            raise RuntimeError("apply_gate: evolved wavefunction vanished")


def _finish_layer(psi: SymmetricMPS, plans, fs, seconds, handle) -> List[GateStats]:
    """mps.cpp:276-321 for every bond: trim, renormalise, lift (one grouped
    product for the layer), gauge update (one table launch for the layer)."""
    torch = _torch()
    h = handle or _lib.default_handle()
    d = psi.site.dim
    p = psi.site.charges
    lift, gauge = _Tables(), _Tables()
    stats, cplx = [], False
    for plan, f in zip(plans, fs):
        factors = f.factors
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
                q = plan.qfac[sp]
                if q is None:
                    continue  # qfac = I: theta' was x y itself
                left = factors[sp].left
                lifted = _colmajor(q.shape[0], left.shape[1], left)
                lift.gemm(lifted, q, left)
                factors[sp].left = lifted
        plan.kept_sq = kept_sq
        cplx = cplx or factors[0].left.is_complex()
    with _lib.on_torch_stream(h):
        lift.run_gemm(h, cplx)
    for plan, f in zip(plans, fs):
        factors = f.factors
        bond = plan.bond
        lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
        inv_norm = 1.0 / np.sqrt(plan.kept_sq)
        for s in (0, 1):
            lam_m[s] = factors[s].sigma * inv_norm
        linv = [_floored_inverse(lam_l[0]), _floored_inverse(lam_l[1])]
        rinv = [_floored_inverse(lam_r[0]), _floored_inverse(lam_r[1])]
        g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
        nl, nr = plan.nl, plan.nr
        for m in range(d):
            for a in (0, 1):
                s = a ^ p[m]
                left = factors[s].left
                lrows = left[plan.row_off[s][m]:plan.row_off[s][m] + nl[a], :]
                g1[m][a] = _colmajor(nl[a], left.shape[1], left)
                gauge.combine(g1[m][a], [(lrows, linv[a], None, 1.0)])
                ra = factors[a].right_adj
                c = a ^ p[m]
                rcols = ra[:, plan.col_off[a][m]:plan.col_off[a][m] + nr[c]]
                g2[m][a] = _colmajor(ra.shape[0], nr[c], ra)
                gauge.combine(g2[m][a], [(rcols, None, rinv[c], 1.0)])
        out = GateStats()
        out.discarded_weight = max(0.0, 1.0 - plan.kept_sq / plan.total_sq)
        out.factorize_seconds = seconds / max(len(plans), 1)
        out.mid_rank = int(lam_m[0].numel() + lam_m[1].numel())
        stats.append(out)
        plan._keep_gauge = (linv, rinv)
    with _lib.on_torch_stream(h):
        gauge.run_combine(h, cplx)
    # the table operands (factors, inverse lambdas) must outlive the launch
    torch.cuda.current_stream().synchronize()
    return stats


def apply_gate(psi: SymmetricMPS, bond: int, gate: TwoSiteGate, chi: int, method: BlockMethod,
               request: Optional[SectorRankRequest] = None, handle=None) -> GateStats:
    """rlftn::apply_gate (mps.cpp:111-323) on device-resident tensors."""
    return apply_gate_layer(psi, [bond], [gate], chi, method, request, handle)[0]


def apply_gate_layer(psi: SymmetricMPS, bonds: Sequence[int], gates: Sequence[TwoSiteGate],
                     chi: int, method: BlockMethod, request: Optional[SectorRankRequest] = None,
                     handle=None) -> List[GateStats]:
    """One TEBD layer: gates on disjoint bonds (mps.cpp:448-457), all theta'
    assembled first (engine table kernels, _assemble_layer), then ONE batched
    block factorization for all bonds (equal-shape sector blocks of different
    bonds share engine calls), then the per-bond trims and one gauge-update
    launch.  Same result as applying the gates one by one."""
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
    plans = [_bond_sizes(psi, b, g) for b, g in zip(bonds, gates)]
    _assemble_layer(psi, plans, handle)
    torch = _torch()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fs = block_factorize_many([BlockDiagMatrix([0, 1], pl.thetap) for pl in plans], chi, request,
                              method, handle)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return _finish_layer(psi, plans, fs, dt, handle)
