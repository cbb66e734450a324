"""Where does the host-pointer (e2e) call spend its time?  C4, 2 chunks."""
import ctypes, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
from paper_1710_01463_b200 import Handle, RsvdParams, _lib, rsvd_batched, synth

cfg = synth.CONFIGS["C4"]
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
h = Handle(0)
Ah = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
Ah.copy_(A)
bsz, m, n = A.shape
k = cfg.rank


def t(f, n=3):
    f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1000


def alloc():
    U = torch.empty((bsz, k, m), dtype=torch.float64, pin_memory=True)
    S = torch.empty((bsz, k), dtype=torch.float64, pin_memory=True)
    V = torch.empty((bsz, n, k), dtype=torch.float64, pin_memory=True)
    return U, S, V


print("wrapper call ms", t(lambda: rsvd_batched(Ah, p, seeds, handle=h)))
print("pinned output alloc ms", t(alloc))
U, S, V = alloc()
lib = _lib.load()
seeds_arr = (ctypes.c_uint64 * bsz)(*seeds)
ranks = (ctypes.c_int64 * bsz)()
dws = (ctypes.c_double * bsz)()


def raw():
    rc = lib.rsvd_f64_batched(h.raw, bsz, Ah.data_ptr(), m, n, m, m * n, p.rank, p.oversample,
                              p.power, seeds_arr, U.data_ptr(), m, m * k, S.data_ptr(), k,
                              V.data_ptr(), k, k * n, ranks, dws, _lib.PTR_HOST)
    assert rc == 0


print("raw C-ABI call ms (preallocated pinned outputs)", t(raw))
Up = torch.empty((bsz, k, m), dtype=torch.float64)
Sp = torch.empty((bsz, k), dtype=torch.float64)
Vp = torch.empty((bsz, n, k), dtype=torch.float64)


def raw_pageable():
    rc = lib.rsvd_f64_batched(h.raw, bsz, Ah.data_ptr(), m, n, m, m * n, p.rank, p.oversample,
                              p.power, seeds_arr, Up.data_ptr(), m, m * k, Sp.data_ptr(), k,
                              Vp.data_ptr(), k, k * n, ranks, dws, _lib.PTR_HOST)
    assert rc == 0


print("raw C-ABI call ms (pageable outputs)", t(raw_pageable))
