"""Synthetic workloads of BASELINE.json's five configurations.

There is no public dataset for this path: BASELINE.json fully specifies the
inputs as A = U diag(sigma) V^T with Haar-random factors (QR of seeded
standard-normal matrices, columns sign-fixed by diag(R)) and closed-form
spectra.  Seeds follow docs/seeds.md (derive_seed = seed ^ mix64(tag)):

  master seed s_c = c for config c = 1..5
  matrix stream   = derive_seed(s_c, 3)  (bench_matrix), item b: derive_seed(., b),
                    factors U/V/g: derive_seed(., 1 / 2 / 3)
  Omega stream    = derive_seed(s_c, 2)  (rsvd_stream),  item b: derive_seed(., b)

Gaussians come from the CounterRng stream (rng.hpp) — on the GPU through the
engine's own generator, on the CPU through a caller-supplied ``gauss``
callable (the tests pass the oracle's).  The QR is torch.linalg.qr on the
chosen device: input generation is test/bench infrastructure, not the timed
path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

from .rng import CounterRng, derive_seed, seed_tag


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    batch: int
    rank: int
    oversample_p: int  # BASELINE's p; the reference's RsvdParams.oversample is rank + p
    power: int
    spectrum: str
    master_seed: int

    @property
    def ell(self) -> int:
        return self.rank + self.oversample_p


CONFIGS = {
    "C1": Config("C1", 1024, 1024, 1, 64, 10, 2, "exp32", 1),
    "C2": Config("C2", 256, 256, 256, 128, 10, 2, "pow1.5", 2),
    "C3": Config("C3", 4096, 4096, 1, 256, 16, 1, "harmonic_gap", 3),
    "C3q3": Config("C3q3", 4096, 4096, 1, 256, 16, 3, "harmonic_gap", 3),
    "C4": Config("C4", 4096, 4096, 32, 256, 20, 2, "exp0.02_noisy", 4),
    "C5": Config("C5", 32768, 2048, 1, 512, 32, 4, "pow0.5", 5),
}


def matrix_seed(cfg: Config, item: int) -> int:
    return derive_seed(derive_seed(cfg.master_seed, seed_tag.bench_matrix), item)


def omega_seed(cfg: Config, item: int) -> int:
    return derive_seed(derive_seed(cfg.master_seed, seed_tag.rsvd_stream), item)


def spectrum(cfg: Config, item: int, count: int, gauss: Callable[[int, int], "object"]):
    """sigma_i for i < count as a python list (descending)."""
    kind = cfg.spectrum
    if kind == "exp32":
        return [math.exp(-i / 32.0) for i in range(count)]
    if kind == "pow1.5":
        s = [(i + 1) ** -1.5 for i in range(count)]
        nrm = math.sqrt(sum(x * x for x in s))
        return [x / nrm for x in s]
    if kind == "harmonic_gap":
        return [(1.0 / (i + 1)) if i < 512 else 1e-8 / (i + 1) for i in range(count)]
    if kind == "exp0.02_noisy":
        g = sorted((float(x) for x in gauss(derive_seed(matrix_seed(cfg, item), 3), count)),
                   reverse=True)
        return [math.exp(-0.02 * i) * (1.0 + 0.1 * g[i]) for i in range(count)]
    if kind == "pow0.5":
        return [(i + 1) ** -0.5 for i in range(count)]
    raise ValueError(kind)


def device_gauss(device):
    """Gaussian CounterRng stream on the GPU via the engine's generator."""
    import torch

    def g(seed: int, count: int):
        out = torch.empty(count, dtype=torch.float64, device=device)
        CounterRng(seed).fill_gaussian(out)
        return out

    return g


def haar_torch(seed: int, rows: int, cols: int, gauss, device):
    """Orthonormal columns from the QR of a seeded Gaussian (column-major
    fill), sign-fixed by diag(R)."""
    import torch

    g = torch.as_tensor(gauss(seed, rows * cols), dtype=torch.float64, device=device)
    g = g.reshape(cols, rows).t()  # column-major rows x cols
    q, r = torch.linalg.qr(g)
    d = torch.sign(torch.diagonal(r))
    d[d == 0] = 1.0
    return q * d[None, :]


def make_matrix(cfg: Config, item: int, device="cuda", gauss: Optional[Callable] = None):
    """A (m x n, float64, column-major strides) for batch item ``item``."""
    import torch

    gauss = gauss or device_gauss(device)
    ms = matrix_seed(cfg, item)
    k = min(cfg.m, cfg.n)
    u = haar_torch(derive_seed(ms, 1), cfg.m, k, gauss, device)
    v = haar_torch(derive_seed(ms, 2), cfg.n, k, gauss, device)
    s = torch.tensor(spectrum(cfg, item, k, gauss), dtype=torch.float64, device=device)
    # A^T = V diag(s) U^T row-major == A column-major.
    at = (v * s[None, :]) @ u.t()
    return at.t()


def make_batch(cfg: Config, device="cuda", batch: Optional[int] = None, first_item: int = 0,
               gauss: Optional[Callable] = None):
    """(batch, m, n) tensor with column-major items (strides (m*n, 1, m))."""
    import torch

    b = cfg.batch if batch is None else batch
    out = torch.empty((b, cfg.n, cfg.m), dtype=torch.float64, device=device)
    for i in range(b):
        out[i] = make_matrix(cfg, first_item + i, device, gauss).t()
    return out.transpose(1, 2)


def omega_seeds(cfg: Config, batch: Optional[int] = None, first_item: int = 0):
    b = cfg.batch if batch is None else batch
    return [omega_seed(cfg, first_item + i) for i in range(b)]
