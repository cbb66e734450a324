"""Row-sharded RSVD on one GPU: P ranks emulated as host threads
with their own handles, joined by an in-process group (host barriers only, no
device-side waits), against the unsharded engine and the oracle."""
import threading

import numpy as np
import pytest

from tests.helpers import isometry_err, matrix_with_spectrum, rel_sigma_err, subspace_distance

pytestmark = pytest.mark.gpu


def run_sharded(A, params, world):
    import torch

    from paper_1710_01463_b200 import Handle, _lib, sharding

    m = A.shape[0]
    group = sharding.Group(world)
    results = [None] * world
    run_sharded.gemm_paths = [None] * world
    errors = []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            h = Handle(0)
            group.attach(h, rank)
            first, count = sharding.row_partition(m, world, rank)
            a_loc = A[first:first + count]
            with torch.cuda.stream(torch.cuda.Stream()):
                f = sharding.rsvd_rowsharded(a_loc, m, first, params, h)
                torch.cuda.synchronize()
            results[rank] = (first, count, f)
            run_sharded.gemm_paths[rank] = _lib.last_gemm_path(h)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]
    return results


@pytest.mark.parametrize("world", [2, 3])
def test_rowsharded_matches_unsharded_and_oracle(cuda, oracle_mod, world, ref_mod):
    import torch

    from paper_1710_01463_b200 import RsvdParams, rsvd

    m, n, k, ell, q, seed = 700, 300, 24, 40, 2, 0xC0FFEE
    a = matrix_with_spectrum(oracle_mod, 99, m, n, np.exp(-np.arange(n) / 25.0))
    A = torch.from_numpy(a).to(cuda).t().contiguous().t()
    p = RsvdParams(k, ell, q, seed)
    res = run_sharded(A, p, world)
    ref = ref_mod.rsvd(a, k, ell, q, seed)
    single = rsvd(A, p)
    U = np.zeros((m, res[0][2].rank()))
    for first, count, f in res:
        assert f.rank() == res[0][2].rank()
        assert torch.equal(f.sigma, res[0][2].sigma)  # replicated parts are identical
        assert torch.equal(f.right_adj, res[0][2].right_adj)
        U[first:first + count] = f.left.cpu().numpy()
    f0 = res[0][2]
    S = f0.sigma.cpu().numpy()
    Vt = f0.right_adj.cpu().numpy()
    assert len(S) == len(ref[1])
    assert rel_sigma_err(S, ref[1]) < 1e-10
    assert rel_sigma_err(S, single.sigma.cpu().numpy()) < 1e-12
    assert isometry_err(U) < 1e-12 and isometry_err(Vt.T) < 1e-12
    e = np.linalg.norm(a - (U * S) @ Vt)
    er = np.linalg.norm(a - (ref[0] * ref[1]) @ ref[2])
    assert abs(e - er) / er < 1e-10
    assert subspace_distance(U[:, :20], ref[0][:, :20]) < 1e-8
    assert f0.discarded_weight == pytest.approx(ref[3], rel=1e-8)


def test_rowsharded_on_the_int8_path(cuda, oracle_mod, ref_mod):
    """Two row shards of a 4096 x 2048 matrix: each rank's 2048 x 2048 shard
    is large enough for the emulated-FP64 A-passes (INT8 tensor cores, per-rank
    row / column exponents of its own shard), the all-reduced A^T Q panels and
    Grams are FP64.  Same tolerances against the reference build."""
    import torch

    from paper_1710_01463_b200 import RsvdParams

    m, n, k, ell, q, seed = 4096, 2048, 256, 276, 1, 0xBEEF
    a = matrix_with_spectrum(oracle_mod, 5, m, n, np.exp(-np.arange(n) / 60.0))
    A = torch.from_numpy(a).to(cuda).t().contiguous().t()
    res = run_sharded(A, RsvdParams(k, ell, q, seed), 2)
    assert run_sharded.gemm_paths == ["ozaki", "ozaki"]
    ref = ref_mod.rsvd(a, k, ell, q, seed)
    f0 = res[0][2]
    U = np.zeros((m, f0.rank()))
    for first, count, f in res:
        assert torch.equal(f.sigma, f0.sigma) and torch.equal(f.right_adj, f0.right_adj)
        U[first:first + count] = f.left.cpu().numpy()
    S, Vt = f0.sigma.cpu().numpy(), f0.right_adj.cpu().numpy()
    assert len(S) == len(ref[1]) == k
    assert rel_sigma_err(S, ref[1]) < 1e-10
    assert isometry_err(U) < 1e-12 and isometry_err(Vt.T) < 1e-12
    e = np.linalg.norm(a - (U * S) @ Vt)
    er = np.linalg.norm(a - (ref[0] * ref[1]) @ ref[2])
    assert abs(e - er) / er < 1e-10
    assert f0.discarded_weight == pytest.approx(ref[3], rel=1e-8)


def test_rowsharded_rank_deficient(cuda, oracle_mod):
    """Completion uses global row indices: a rank-5 matrix still factors."""
    import torch

    from paper_1710_01463_b200 import RsvdParams

    m, n = 200, 120
    a = matrix_with_spectrum(oracle_mod, 7, m, n, [5.0, 4.0, 3.0, 2.0, 1.0])
    A = torch.from_numpy(a).to(cuda).t().contiguous().t()
    res = run_sharded(A, RsvdParams(10, 20, 2, 5), 2)
    f0 = res[0][2]
    assert f0.rank() == 5
    U = np.zeros((m, 5))
    for first, count, f in res:
        U[first:first + count] = f.left.cpu().numpy()
    rec = (U * f0.sigma.cpu().numpy()) @ f0.right_adj.cpu().numpy()
    assert np.linalg.norm(a - rec) <= 1e-10 * np.linalg.norm(a)


def test_rowsharded_requires_communicator(cuda):
    import torch

    from paper_1710_01463_b200 import Handle, InvalidArgument, RsvdParams, sharding

    h = Handle(0)
    A = torch.randn(64, 32, dtype=torch.float64, device=cuda).t().contiguous().t()
    with pytest.raises(InvalidArgument, match="no group"):
        sharding.rsvd_rowsharded(A, 128, 0, RsvdParams(4, 8, 1, 1), h)
