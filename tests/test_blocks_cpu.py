"""Block (symmetry-sector) factorization: host logic and the oracle, no GPU.

Restates proj/tests/test_blocks.cpp against (a) the product's host-side
`sector_request` and argument checks and (b) the oracle's block_factorize
restatement (oracle/rsvd_oracle.cpp, blocks.cpp:38-118), pinning the oracle
before it is used as the GPU checker in test_gpu_blocks.py.
"""
import numpy as np
import pytest

from paper_1710_01463_b200 import blocks as B
from paper_1710_01463_b200._lib import InvalidArgument

from .helpers import matrix_with_spectrum, spectrum_family


def _req(chi, slack=-1, maximal=False):
    return B.SectorRankRequest(B.RankPolicy.maximal if maximal else B.RankPolicy.per_sector_estimate,
                               chi, slack)


def test_sector_request_base_plus_slack():  # test_blocks.cpp:42-63
    assert B.sector_request(_req(100, 2), [60, 60]) == [52, 52]
    assert B.sector_request(_req(10, 2), [100]) == [12]
    assert B.sector_request(_req(100), [60, 60]) == [53, 53]
    assert B.sector_request(_req(10), [100, 100]) == [7, 7]
    assert B.sector_request(_req(100, 2), [20, 60]) == [20, 52]


def test_sector_request_maximal():  # test_blocks.cpp:65-72
    assert B.sector_request(_req(100, maximal=True), [80, 30]) == [80, 30]
    assert B.sector_request(_req(10, maximal=True), [80, 30]) == [10, 10]


def test_sector_request_invalid():  # test_blocks.cpp:74-80
    with pytest.raises(InvalidArgument, match="chi must be >= 1"):
        B.sector_request(_req(0), [10])
    with pytest.raises(InvalidArgument, match="at least one sector"):
        B.sector_request(_req(5), [])


@pytest.mark.parametrize("chi,slack,maximal,dims", [
    (100, 2, False, [60, 60]), (10, -1, False, [100, 100]), (37, -1, False, [5, 40, 17]),
    (400, -1, False, [100] * 7), (10, 0, True, [80, 3, 0]), (1, -1, False, [1]),
])
def test_sector_request_matches_oracle(oracle_mod, chi, slack, maximal, dims):
    assert B.sector_request(_req(chi, slack, maximal), dims) == \
        list(oracle_mod.sector_request(maximal, chi, slack, dims))


def test_block_factorize_input_errors():  # test_blocks.cpp:245-258 (host-side checks)
    m = B.BlockMethod.deterministic()
    with pytest.raises(InvalidArgument, match="no sectors"):
        B.block_factorize(B.BlockDiagMatrix([], []), 2, _req(0), m)
    with pytest.raises(InvalidArgument, match="duplicate sector charge"):
        B.block_factorize(B.BlockDiagMatrix([0, 0], [np.eye(2), np.eye(2)]), 2, _req(0), m)
    with pytest.raises(InvalidArgument, match="size mismatch"):
        B.block_factorize(B.BlockDiagMatrix([0, 1], [np.eye(2)]), 2, _req(0), m)


# ---------------------------------------------------------------- oracle ---

def _two_diag():
    return [np.diag([3.0, 1.0]), np.diag([2.0, 0.5])], [0, 1]


def test_oracle_global_selection(oracle_mod):  # test_blocks.cpp:82-95
    blocks, ch = _two_diag()
    f, dw, exact = oracle_mod.block_factorize(blocks, ch, 2, maximal=True)
    assert [len(x[1]) for x in f] == [1, 1]
    assert f[0][1][0] == pytest.approx(3.0, rel=1e-14)
    assert f[1][1][0] == pytest.approx(2.0, rel=1e-14)
    assert dw == pytest.approx(1.25, rel=1e-14)
    assert exact


def test_oracle_order_independent(oracle_mod):  # test_blocks.cpp:97-112
    blocks, ch = _two_diag()
    fa, _, _ = oracle_mod.block_factorize(blocks, ch, 3, maximal=True)
    fb, _, _ = oracle_mod.block_factorize(blocks[::-1], ch[::-1], 3, maximal=True)
    merged = lambda f: sorted(np.concatenate([x[1] for x in f]), reverse=True)  # noqa: E731
    assert merged(fa) == merged(fb)
    assert len(fa[0][1]) == len(fb[1][1]) and len(fa[1][1]) == len(fb[0][1])


def test_oracle_ties_to_lower_charge(oracle_mod):  # test_blocks.cpp:114-140
    even = np.diag([2.0, 1.0])
    odd = np.diag([2.0, 1.0])
    f, _, _ = oracle_mod.block_factorize([even, odd], [0, 1], 3, maximal=True)
    assert [len(x[1]) for x in f] == [2, 1]
    g, _, _ = oracle_mod.block_factorize([odd, even], [1, 0], 3, maximal=True)
    assert [len(x[1]) for x in g] == [1, 2]


def test_oracle_dense_embedding(oracle_mod):  # test_blocks.cpp:158-183
    rng = np.random.default_rng(33)
    b0 = rng.standard_normal((18, 14))
    b1 = rng.standard_normal((16, 20))
    dense = np.zeros((34, 34))
    dense[:18, :14] = b0
    dense[18:, 14:] = b1
    f, dw, _ = oracle_mod.block_factorize([b0, b1], [0, 1], 9, maximal=True)
    _, st, _, dwt = oracle_mod.tsvd(dense, 9)
    merged = np.sort(np.concatenate([x[1] for x in f]))[::-1]
    assert len(merged) == len(st)
    np.testing.assert_allclose(merged, st, rtol=1e-12)
    assert dw == pytest.approx(dwt, rel=1e-10)


def test_oracle_randomized_matches_deterministic(oracle_mod):  # test_blocks.cpp:185-203
    b0 = matrix_with_spectrum(oracle_mod, 8, 64, 48, spectrum_family(0, 40))
    b1 = matrix_with_spectrum(oracle_mod, 9, 56, 60, spectrum_family(2, 40))
    fd, _, ed = oracle_mod.block_factorize([b0, b1], [0, 1], 24)
    fr, _, er = oracle_mod.block_factorize([b0, b1], [0, 1], 24, kind="rsvd", power=4, seed=2024)
    assert ed and not er
    sd = np.sort(np.concatenate([x[1] for x in fd]))[::-1]
    sr = np.sort(np.concatenate([x[1] for x in fr]))[::-1]
    assert len(sd) == len(sr)
    assert np.max(np.abs(sr - sd) / sd) < 1e-8


def test_oracle_seed_derivation(oracle_mod):  # test_blocks.cpp:222-243
    blk = matrix_with_spectrum(oracle_mod, 44, 64, 64, spectrum_family(2, 50))
    f, _, _ = oracle_mod.block_factorize([blk], [1], 10, maximal=True, kind="rsvd", power=4,
                                         seed=99, min_dim=1)
    U, S, _, _ = oracle_mod.rsvd(blk, 10, 20, 4, oracle_mod.derive_seed(99, 1))
    assert np.array_equal(f[0][1], S) and np.array_equal(f[0][0], U)


def test_oracle_oversample_clamped(oracle_mod):  # test_blocks.cpp:224-243
    blk = np.random.default_rng(50).standard_normal((40, 36))
    for ov in (4, 500):
        f, _, _ = oracle_mod.block_factorize([blk], [0], 12, maximal=True, kind="rsvd", power=2,
                                             seed=7, min_dim=1, oversample=ov)
        assert len(f[0][1]) == 12


def test_oracle_rank_zero_sector(oracle_mod):  # test_blocks.cpp:260-279
    f, dw, _ = oracle_mod.block_factorize([np.diag([9.0, 8.0, 7.0]), np.diag([0.2, 0.1])], [0, 1],
                                          3, maximal=True)
    assert [len(x[1]) for x in f] == [3, 0]
    assert f[1][0].shape == (2, 0)
    assert dw == pytest.approx(0.05, rel=1e-12)
