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


class _BondPlan:
    """Everything the update of one bond needs between its assembly and its
    gauge update (sector offsets, the assembled theta', QR factors)."""


def _colmajor(rows: int, cols: int, like):
    """Uninitialised device matrix in column-major storage (the engine's
    layout; the table kernels write it row-fastest, i.e. coalesced)."""
    torch = _torch()
    return torch.empty((cols, rows), dtype=like.dtype, device=like.device).t()


class _Blk:
    """A strided matrix by address -- (ptr, row stride, column stride, rows,
    cols) in elements -- and the tensor owning its storage.  Sub-blocks are
    address arithmetic, so building the launch tables creates no torch views
    (a view costs microseconds of host time; a layer builds thousands)."""

    __slots__ = ("p", "rs", "cs", "r", "c", "owner", "es")

    def __init__(self, p, rs, cs, r, c, owner, es):
        self.p, self.rs, self.cs, self.r, self.c, self.owner, self.es = p, rs, cs, r, c, owner, es

    @staticmethod
    def of(t):
        return _Blk(t.data_ptr(), t.stride(0), t.stride(1), t.shape[0], t.shape[1], t,
                    t.element_size())

    def sub(self, r0, r1, c0, c1):
        return _Blk(self.p + (r0 * self.rs + c0 * self.cs) * self.es, self.rs, self.cs, r1 - r0,
                    c1 - c0, self.owner, self.es)


class _Arena:
    """One device allocation carved into column-major matrices (the layer's
    intermediate operands)."""

    def __init__(self, total, like):
        torch = _torch()
        self.buf = torch.empty(max(int(total), 1), dtype=like.dtype, device=like.device)
        self.base = self.buf.data_ptr()
        self.es = self.buf.element_size()
        self.off = 0

    def take(self, rows, cols):
        b = _Blk(self.base + self.off * self.es, 1, max(rows, 1), rows, cols, self.buf, self.es)
        self.off += rows * cols
        return b


class _Tables:
    """Host job tables of one launch of the engine's table-driven bond-update
    kernels (rsvd_combine_blocks / rsvd_grouped_gemm / rsvd_block_sqnorms)."""

    def __init__(self):
        self.jobs, self.terms, self.gemms = [], [], []
        self.keep = []  # tensors whose storage the tables point to

    def combine(self, dst, terms):
        """dst = sum_t coef * diag(row_scale) src diag(col_scale); dst and the
        sources are _Blk, terms = [(src, row_scale_ptr or 0, col_scale_ptr or 0,
        coef)]."""
        if dst.r == 0 or dst.c == 0:
            return
        begin = len(self.terms)
        for src, rsc, csc, coef in terms:
            if coef == 0:
                continue
            c = complex(coef)
            self.terms.append((src.p, src.rs, src.cs, rsc, csc, c.real, c.imag))
            self.keep.append(src.owner)
        self.jobs.append((dst.p, dst.rs, dst.cs, dst.r, dst.c, begin, len(self.terms) - begin))
        self.keep.append(dst.owner)

    def gemm(self, c, a, b):
        if c.r == 0 or c.c == 0:
            return
        if a.c == 0:
            self.combine(c, [])
            return
        self.gemms.append((a.p, a.rs, a.cs, b.p, b.rs, b.cs, c.p, c.rs, c.cs, c.r, c.c, a.c))
        self.keep += [a.owner, b.owner, c.owner]

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


def _ptr(t):
    return t.data_ptr() if t is not None else 0


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
    # One allocation for every block-form intermediate (A_mu, B_mu, theta_mu)
    # of the layer, and the theta' outputs (handed to the factorization as
    # tensors) carved from a second one.
    need = 0
    need_out = 0
    for pl in plans:
        if pl.gate.form == GateForm.block:
            for mu in (0, 1):
                if pl.nm[mu]:
                    need += pl.rows[mu] * pl.nm[mu] + pl.nm[mu] * pl.cols[mu] + \
                        pl.rows[mu] * pl.cols[mu]
            need_out += pl.rows[0] * pl.cols[0] + pl.rows[1] * pl.cols[1]
    arena = _Arena(need, ref)
    outbuf = torch.empty(max(need_out, 1), dtype=ref.dtype, device=dev)
    out_off = 0
    blk_cache = {}

    def blk(t):  # _Blk of a state tensor, cached for the layer
        k = id(t)
        v = blk_cache.get(k)
        if v is None:
            v = _Blk.of(t)
            blk_cache[k] = v
        return v

    for pl in plans:
        bond = pl.bond
        lam_l, lam_m, lam_r = psi.lambdas[bond], psi.lambdas[bond + 1], psi.lambdas[bond + 2]
        g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
        nl, nm, nr, rows, cols = pl.nl, pl.nm, pl.nr, pl.rows, pl.cols
        row_off, col_off = pl.row_off, pl.col_off
        gate = pl.gate
        if gate.form == GateForm.block:
            pl.lifted = False
            theta = [None, None]
            pll = [_ptr(lam_l[0]), _ptr(lam_l[1])]
            plm = [_ptr(lam_m[0]), _ptr(lam_m[1])]
            plr = [_ptr(lam_r[0]), _ptr(lam_r[1])]
            for mu in (0, 1):
                if nm[mu] == 0:
                    continue
                A = arena.take(rows[mu], nm[mu])
                B = arena.take(nm[mu], cols[mu])
                for m in range(d):
                    a = mu ^ p[m]
                    st1.combine(A.sub(row_off[mu][m], row_off[mu][m] + nl[a], 0, nm[mu]),
                                [(blk(g1[m][a]), pll[a], plm[mu], 1.0)])
                    st1.combine(B.sub(0, nm[mu], col_off[mu][m], col_off[mu][m] + nr[a]),
                                [(blk(g2[m][mu]), 0, plr[a], 1.0)])
                theta[mu] = arena.take(rows[mu], cols[mu])
                st2.gemm(theta[mu], A, B)
            gb = gate.block
            thetap, tpb = [], []
            for sp in (0, 1):
                n_ = rows[sp] * cols[sp]
                t_ = outbuf.narrow(0, out_off, n_).view(cols[sp], rows[sp]).t()
                out_off += n_
                thetap.append(t_)
                tpb.append(_Blk(t_.data_ptr(), 1, max(rows[sp], 1), rows[sp], cols[sp], outbuf,
                                arena.es))
            for sp in (0, 1):
                for m1 in range(d):
                    a = sp ^ p[m1]
                    for m2 in range(d):
                        c = sp ^ p[m2]
                        q = p[m1] ^ p[m2]
                        out = tpb[sp].sub(row_off[sp][m1], row_off[sp][m1] + nl[a],
                                          col_off[sp][m2], col_off[sp][m2] + nr[c])
                        terms = []
                        for i1 in range(d):
                            for i2 in range(d):
                                if p[i1] ^ p[i2] != q:
                                    continue
                                coef = float(gb[m1 * d + m2, i1 * d + i2])
                                mu = a ^ p[i1]
                                if coef == 0.0 or theta[mu] is None:
                                    continue
                                src = theta[mu].sub(row_off[mu][i1], row_off[mu][i1] + nl[a],
                                                    col_off[mu][i2], col_off[mu][i2] + nr[c])
                                terms.append((src, 0, 0, coef))
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
                xb, yb = _Blk.of(x), _Blk.of(y)
                for k, t in enumerate(gate.terms):
                    mu = sp ^ t.charge
                    w = nm[mu]
                    if w == 0:
                        continue
                    for m1p in range(d):
                        a = sp ^ p[m1p]
                        st1.combine(xb.sub(row_off[sp][m1p], row_off[sp][m1p] + nl[a],
                                           koff[k], koff[k] + w),
                                    [(blk(g1[m1][a]), _ptr(lam_l[a]), _ptr(lam_m[mu]),
                                      float(t.left[m1p, m1]))
                                     for m1 in range(d) if t.left[m1p, m1] != 0.0])
                    for m2p in range(d):
                        c = sp ^ p[m2p]
                        st1.combine(yb.sub(koff[k], koff[k] + w,
                                           col_off[sp][m2p], col_off[sp][m2p] + nr[c]),
                                    [(blk(g2[m2][mu]), 0, _ptr(lam_r[c]), float(t.right[m2p, m2]))
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
                st2.gemm(_Blk.of(pl.thetap[sp]), _Blk.of(Rb[i]), _Blk.of(y))
        for pl, sp, x, y in lifted_y:
            st2.gemm(_Blk.of(pl.thetap[sp]), _Blk.of(x), _Blk.of(y))
        # (2) theta_mu = Astack Bstack, R y, x y
        st2.run_gemm(h, cplx)
        # (3) gate mixing
        st3.run_combine(h, cplx)
        # (4) ||theta'||^2 per bond, one device -> host transfer for the layer
        blocks, begin = [], [0]
        for pl in plans:
            for tp in pl.thetap:
                if tp is not None and tp.numel():
                    blocks.append((tp.data_ptr(), tp.stride(0), tp.stride(1), tp.shape[0],
                                   tp.shape[1], 0, 0))
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
        pl._keep = (st1.keep, st2.keep, st3.keep, arena)
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
                lift.gemm(_Blk.of(lifted), _Blk.of(q), _Blk.of(left))
                factors[sp].left = lifted
        plan.kept_sq = kept_sq
        plan.sig_host = sh
        cplx = cplx or factors[0].left.is_complex()
    with _lib.on_torch_stream(h):
        lift.run_gemm(h, cplx)
    # 1 / max(lambda, floor) of every outer bond of the layer in one pass (the
    # outer bonds of disjoint gates are not updated by this layer)
    outer = []
    for plan in plans:  # (plans is never empty: apply_gate_layer takes >= 1 bond)
        outer += [psi.lambdas[plan.bond][0], psi.lambdas[plan.bond][1],
                  psi.lambdas[plan.bond + 2][0], psi.lambdas[plan.bond + 2][1]]
    inv_all = torch.split(1.0 / torch.clamp(torch.cat(outer), min=LAMBDA_FLOOR),
                          [t.numel() for t in outer])
    # The new inner lambdas sigma / ||kept|| of the whole layer from the host
    # copies of sigma, uploaded in one transfer (the same IEEE products).
    lam_vals, lam_dst = [], []
    # The new Gamma blocks of the layer: one allocation, column-major blocks.
    gsize = 0
    for plan, f in zip(plans, fs):
        for m in range(d):
            for a in (0, 1):
                gsize += plan.nl[a] * f.factors[a ^ p[m]].left.shape[1]
                gsize += f.factors[a].right_adj.shape[0] * plan.nr[a ^ p[m]]
    like = fs[0].factors[0].left
    garena = torch.empty(max(gsize, 1), dtype=like.dtype, device=like.device)
    goff = 0

    def gtake(rows, cols):
        nonlocal goff
        n_ = rows * cols
        t_ = garena.narrow(0, goff, n_).view(cols, rows).t()
        goff += n_
        return t_

    for pi, (plan, f) in enumerate(zip(plans, fs)):
        factors = f.factors
        bond = plan.bond
        lam_m = psi.lambdas[bond + 1]
        inv_norm = 1.0 / np.sqrt(plan.kept_sq)
        for s in (0, 1):
            lam_vals.append(np.asarray(plan.sig_host[s], dtype=np.float64) * inv_norm)
            lam_dst.append((lam_m, s))
        linv = inv_all[4 * pi:4 * pi + 2]
        rinv = inv_all[4 * pi + 2:4 * pi + 4]
        pli = [_ptr(linv[0]), _ptr(linv[1])]
        pri = [_ptr(rinv[0]), _ptr(rinv[1])]
        g1, g2 = psi.gammas[bond], psi.gammas[bond + 1]
        nl, nr = plan.nl, plan.nr
        lb = [_Blk.of(factors[0].left), _Blk.of(factors[1].left)]
        rb = [_Blk.of(factors[0].right_adj), _Blk.of(factors[1].right_adj)]
        for m in range(d):
            for a in (0, 1):
                s = a ^ p[m]
                L = lb[s]
                g1[m][a] = gtake(nl[a], L.c)
                gauge.combine(_Blk.of(g1[m][a]),
                              [(L.sub(plan.row_off[s][m], plan.row_off[s][m] + nl[a], 0, L.c),
                                pli[a], 0, 1.0)])
                R = rb[a]
                c = a ^ p[m]
                g2[m][a] = gtake(R.r, nr[c])
                gauge.combine(_Blk.of(g2[m][a]),
                              [(R.sub(0, R.r, plan.col_off[a][m], plan.col_off[a][m] + nr[c]), 0,
                                pri[c], 1.0)])
        out = GateStats()
        out.discarded_weight = max(0.0, 1.0 - plan.kept_sq / plan.total_sq)
        out.factorize_seconds = seconds / max(len(plans), 1)
        out.mid_rank = int(len(plan.sig_host[0]) + len(plan.sig_host[1]))  # the new lambdas
        stats.append(out)
        plan._keep_gauge = (linv, rinv, inv_all)
    allv = torch.from_numpy(np.concatenate(lam_vals)).to(like.device)
    for (lst, s_), piece in zip(lam_dst, torch.split(allv, [len(v) for v in lam_vals])):
        lst[s_] = piece
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
