"""Multi-process (gloo, world_size 2, CPU) checks of the multi-GPU
decomposition:

* the batch split and row partition helpers used by bench.py;
* the row-sharded algebra of engine.cu — Omega replicated from the seed,
  Y_p = A_p Omega local, Grams and A^T Q panels sum-all-reduced, n-side
  orthonormalisation and the small SVD replicated, U_p = Q_p U~ local —
  restated in numpy over torch.distributed(gloo) and checked against the
  oracle's unsharded rsvd on the same Omega."""
import os
import socket

import numpy as np
import pytest


def test_batch_partition_covers_everything():
    from paper_1710_01463_b200.sharding import batch_partition

    for batch in (1, 7, 32, 256):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, count = batch_partition(batch, world, r)
                seen.extend(range(first, first + count))
            assert seen == list(range(batch))


def test_row_partition_aligned_and_complete():
    from paper_1710_01463_b200.sharding import row_partition

    for m in (200, 4096, 32768, 1000):
        for world in (1, 2, 4, 8):
            rows = []
            for r in range(world):
                first, count = row_partition(m, world, r)
                if count:
                    assert first % 16 == 0
                rows.extend(range(first, first + count))
            assert rows == list(range(m))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_1710_01463_b200.sharding import row_partition
    from tests.helpers import matrix_with_spectrum

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    m, n, k, ell, q, seed = 360, 200, 16, 28, 2, 4321
    a = matrix_with_spectrum(oracle, 5, m, n, np.exp(-np.arange(n) / 18.0))
    first, count = row_partition(m, world, rank)
    A_p = a[first:first + count]
    om = oracle.gaussian_matrix(seed, n, ell)  # replicated from the seed

    def orth_m(Y, passes):
        for _ in range(passes):  # CholeskyQR with an all-reduced Gram
            G = allreduce(Y.T @ Y)
            R = np.linalg.cholesky(G).T
            Y = np.linalg.solve(R.T, Y.T).T
        return Y

    Q = orth_m(A_p @ om, 1 if q else 2)
    for t in range(q):
        Z = allreduce(A_p.T @ Q)
        Qz = np.linalg.qr(Z)[0]
        Q = orth_m(A_p @ Qz, 2 if t + 1 == q else 1)
    Bt = allreduce(A_p.T @ Q)
    Ub, s, Vbt = np.linalg.svd(Bt.T, full_matrices=False)
    cut = max(m, n) * np.finfo(float).eps * s[0]
    r = min(k, int(np.sum(s > cut)))
    U_p = Q @ Ub[:, :r]
    np.save(os.path.join(out_dir, f"u{rank}.npy"), U_p)
    if rank == 0:
        np.save(os.path.join(out_dir, "s.npy"), s[:r])
        np.save(os.path.join(out_dir, "vt.npy"), Vbt[:r])
        np.save(os.path.join(out_dir, "a.npy"), a)
    dist.barrier()
    dist.destroy_process_group()


def test_rowsharded_algebra_gloo_world2(tmp_path, oracle_mod):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_sharded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    a = np.load(tmp_path / "a.npy")
    s = np.load(tmp_path / "s.npy")
    vt = np.load(tmp_path / "vt.npy")
    U = np.concatenate([np.load(tmp_path / f"u{r}.npy") for r in range(world)])
    Ur, Sr, Vtr, _ = oracle_mod.rsvd(a, 16, 28, 2, 4321)
    assert len(s) == len(Sr)
    assert np.max(np.abs(s - Sr) / Sr) < 1e-10
    e = np.linalg.norm(a - (U * s) @ vt)
    er = np.linalg.norm(a - (Ur * Sr) @ Vtr)
    assert abs(e - er) / er < 1e-10
