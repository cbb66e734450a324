"""Block-diagonal (symmetry-sector) factorization on the GPU engine.

Mirrors rlftn's blocks.hpp / blocks.cpp (proj/include/rlftn/blocks.hpp:49-63,
proj/src/blocks.cpp:19-118): the caller of the RSVD path in a TEBD bond update
(mps.cpp:275-277).  Per sector: rsvd when `kind == rsvd` and
min(m, n) >= rsvd_min_dim (blocks.cpp:69-70) with rank = the sector request,
the sample width clamped to [want, dim] (or 2 * want, clipped; blocks.cpp:76-77)
and seed derive_seed(base seed, charge) (blocks.cpp:78); tsvd otherwise
(blocks.cpp:82).  Sectors with equal shapes and parameters are factorized in
one batched engine call.  Then the global top-chi post-selection with ties
broken by (charge asc, position asc) (blocks.cpp:86-105) and the trim with
discarded weights (blocks.cpp:107-116).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field, replace
from typing import Any, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import InvalidArgument
from .factorize import (RsvdParams, TruncatedFactorization, _is_torch_cuda, rsvd, rsvd_batched,
                        tsvd, tsvd_batched)
from .rng import derive_seed


class RankPolicy(enum.Enum):
    per_sector_estimate = 0  # chi'_s = ceil(chi / N) + slack, clipped to the block
    maximal = 1              # chi'_s = min(chi, block dimension)


@dataclass
class SectorRankRequest:
    policy: RankPolicy = RankPolicy.per_sector_estimate
    chi: int = 0
    slack: int = -1  # < 0: max(2, ceil(0.05 * chi / N))


@dataclass
class BlockMethod:
    kind: str = "tsvd"  # "tsvd" | "rsvd"
    rsvd: RsvdParams = field(default_factory=RsvdParams)
    rsvd_min_dim: int = 32

    @staticmethod
    def deterministic() -> "BlockMethod":
        return BlockMethod()

    @staticmethod
    def randomized(power: int = 4, seed: int = 0) -> "BlockMethod":
        return BlockMethod("rsvd", RsvdParams(0, 0, power, seed))


@dataclass
class BlockDiagMatrix:
    charges: List[int]
    blocks: List[Any]

    def sector_count(self) -> int:
        return len(self.blocks)


@dataclass
class BlockFactorization:
    charges: List[int]
    factors: List[TruncatedFactorization]
    discarded_weight: float = 0.0
    discarded_exact: bool = True

    def total_rank(self) -> int:
        return sum(f.rank() for f in self.factors)


def _ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


def sector_request(request: SectorRankRequest, block_dims: Sequence[int]) -> List[int]:
    """blocks.cpp:19-36."""
    if request.chi < 1:
        raise InvalidArgument("sector_request: chi must be >= 1")
    n = len(block_dims)
    if n < 1:
        raise InvalidArgument("sector_request: need at least one sector")
    if request.policy == RankPolicy.maximal:
        return [min(request.chi, d) for d in block_dims]
    base = _ceil_div(request.chi, n)
    slack = request.slack if request.slack >= 0 else max(2, _ceil_div(base, 20))
    return [min(base + slack, d) for d in block_dims]


def _shape(b) -> Tuple[int, int]:
    return int(b.shape[0]), int(b.shape[1])


def _sqnorm(b) -> float:
    if _is_torch_cuda(b):
        return float((b.abs() ** 2).sum().item()) if b.is_complex() else float((b * b).sum().item())
    x = np.asarray(b)
    return float(np.sum(np.abs(x) ** 2)) if np.iscomplexobj(x) else float(
        np.sum(np.asarray(x, dtype=np.float64) ** 2))


def _empty_factor(b) -> TruncatedFactorization:
    m, n = _shape(b)
    if _is_torch_cuda(b):
        import torch

        z = lambda *s: torch.zeros(s, dtype=b.dtype, device=b.device)  # noqa: E731
        return TruncatedFactorization(z(m, 0), torch.zeros(0, dtype=torch.float64, device=b.device),
                                      z(0, n), _sqnorm(b), True)
    dt = np.complex128 if np.iscomplexobj(b) else np.float64
    return TruncatedFactorization(np.zeros((m, 0), dtype=dt), np.zeros(0), np.zeros((0, n), dtype=dt),
                                  _sqnorm(b), True)


def _stack(blocks: List[Any]):
    if _is_torch_cuda(blocks[0]):
        import torch

        return torch.stack([x.t() for x in blocks]).transpose(1, 2)  # column-major items
    dt = np.complex128 if any(np.iscomplexobj(x) for x in blocks) else np.float64
    return np.stack([np.asarray(x, dtype=dt) for x in blocks])


def _validate(a: BlockDiagMatrix) -> None:
    if len(a.blocks) != len(a.charges):
        raise InvalidArgument("block_factorize: charges/blocks size mismatch")
    if not a.blocks:
        raise InvalidArgument("block_factorize: no sectors")
    if len(set(a.charges)) != len(a.charges):
        raise InvalidArgument("block_factorize: duplicate sector charge")


def block_factorize_many(mats: Sequence[BlockDiagMatrix], chi: int, request: SectorRankRequest,
                         method: BlockMethod, handle: Optional[_lib.Handle] = None
                         ) -> List[BlockFactorization]:
    """block_factorize of several block-diagonal matrices (e.g. the bonds of
    one TEBD layer) with their sector blocks pooled: every group of equal
    (route, shape, rank, sample width) blocks -- across matrices -- is one
    engine call.  Per matrix the result equals block_factorize."""
    for a in mats:
        _validate(a)
    req = replace(request, chi=chi)
    plans = []  # per matrix: (dims, want)
    factors: List[List[Optional[TruncatedFactorization]]] = []
    exact = []
    groups: Dict[tuple, List[Tuple[int, int]]] = {}
    for mi, a in enumerate(mats):
        dims = [min(_shape(b)) for b in a.blocks]
        want = sector_request(req, dims)
        plans.append((dims, want))
        factors.append([None] * len(a.blocks))
        exact.append(True)
        for s in range(len(a.blocks)):
            if want[s] == 0 or dims[s] == 0:
                factors[mi][s] = _empty_factor(a.blocks[s])
                continue
            m, n = _shape(a.blocks[s])
            dev = str(a.blocks[s].device) if _is_torch_cuda(a.blocks[s]) else "host"
            if method.kind == "rsvd" and dims[s] >= method.rsvd_min_dim:
                ov = method.rsvd.oversample
                ell = min(max(ov, want[s]), dims[s]) if ov > 0 else min(2 * want[s], dims[s])
                key = ("rsvd", dev, m, n, want[s], ell, method.rsvd.power)
                exact[mi] = False
            else:
                key = ("tsvd", dev, m, n, want[s])
            groups.setdefault(key, []).append((mi, s))

    # Host copies of the singular values (the selection runs on the host): one
    # transfer per engine call instead of one per sector.
    host_sig: Dict[Tuple[int, int], np.ndarray] = {}
    for mi, a in enumerate(mats):
        for s, f in enumerate(factors[mi]):
            if f is not None:
                host_sig[(mi, s)] = np.zeros(0)
    for key, members in groups.items():
        blocks = [mats[mi].blocks[s] for mi, s in members]
        if key[0] == "tsvd":
            k = key[4]
            if len(members) == 1:
                mi, s = members[0]
                factors[mi][s] = tsvd(blocks[0], k, handle)
                host_sig[(mi, s)] = _host(factors[mi][s].sigma)
                continue
            bf = tsvd_batched(_stack(blocks), k, handle)
        else:
            _, _, m, n, k, ell, power = key
            seeds = [derive_seed(method.rsvd.seed, int(mats[mi].charges[s])) for mi, s in members]
            if len(members) == 1:
                mi, s = members[0]
                factors[mi][s] = rsvd(blocks[0], RsvdParams(k, ell, power, seeds[0]), handle)
                host_sig[(mi, s)] = _host(factors[mi][s].sigma)
                continue
            bf = rsvd_batched(_stack(blocks), RsvdParams(k, ell, power, 0), seeds, handle)
        sig_all = _host(bf.sigma)
        for i, (mi, s) in enumerate(members):
            factors[mi][s] = bf.item(i)
            host_sig[(mi, s)] = sig_all[i][:bf.ranks[i]]

    return [_select(mats[mi], factors[mi], chi, exact[mi],
                    [host_sig[(mi, s)] for s in range(len(factors[mi]))])
            for mi in range(len(mats))]


def _host(x) -> np.ndarray:
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _select(a: BlockDiagMatrix, factors, chi: int, exact: bool,
            host_sigs=None) -> BlockFactorization:
    """Global post-selection (blocks.cpp:86-116): the chi largest values over
    all sectors, ties to the lower charge then the lower in-sector position;
    dropped values move into the sector's discarded weight.  Each kept factor
    carries `sigma_host`, a host copy of its values."""
    nsec = len(factors)
    cand = []
    sigs = []
    for s, f in enumerate(factors):
        sig = host_sigs[s] if host_sigs is not None else _host(f.sigma)
        sigs.append(sig)
        for pos in range(f.rank()):
            cand.append((-float(sig[pos]), int(a.charges[s]), pos, s))
    cand.sort()
    keep = [0] * nsec
    for c in cand[:chi]:
        keep[c[3]] += 1
    total_dw = 0.0
    out = []
    for s, f in enumerate(factors):
        dw = f.discarded_weight + float(np.sum(sigs[s][keep[s]:] ** 2))
        tf = TruncatedFactorization(f.left[:, :keep[s]], f.sigma[:keep[s]],
                                    f.right_adj[:keep[s], :], dw, f.discarded_exact)
        tf.sigma_host = sigs[s][:keep[s]]
        out.append(tf)
        total_dw += dw
    return BlockFactorization(list(a.charges), out, total_dw, exact)


def block_factorize(a: BlockDiagMatrix, chi: int, request: SectorRankRequest,
                    method: BlockMethod, handle: Optional[_lib.Handle] = None
                    ) -> BlockFactorization:
    """rlftn::block_factorize (blocks.cpp:38-118) on the GPU engine: per-sector
    rsvd / tsvd dispatch (blocks.cpp:60-84; equal-shape sectors share one
    batched engine call), then the global top-chi selection."""
    return block_factorize_many([a], chi, request, method, handle)[0]
