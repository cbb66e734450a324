"""GPU parity of the RSVD path against the CPU oracle (restated reference).

Tolerances (BASELINE.json north_star): singular values 1e-10 relative,
reconstruction error 1e-10 relative, subspace distance <= 1e-8 for gapped
spectra; factor isometry 1e-12 (test_factorize.cpp:73-83)."""
import numpy as np
import pytest

from tests.helpers import (isometry_err, matrix_with_spectrum, rel_sigma_err, spectrum_family,
                           subspace_distance)

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
REC_TOL = 1e-10
SUB_TOL = 1e-8
ISO_TOL = 1e-12


def _gapped_prefix(S, k, rel_gap=1e-3):
    """Largest j <= k such that sigma_{j-1} - sigma_j is a relative gap: the
    leading j-dimensional subspace is well defined."""
    for j in range(min(k, len(S) - 1), 0, -1):
        if (S[j - 1] - S[j]) > rel_gap * S[0]:
            return j
    return 0


def check_against(a, f, ref, label=""):
    from paper_1710_01463_b200 import reconstruction_error

    U, S, Vt, dw = ref
    assert f.rank() == len(S), (label, f.rank(), len(S))
    assert rel_sigma_err(f.sigma, S) < SIG_TOL, label
    left = np.asarray(f.left)
    right = np.asarray(f.right_adj)
    assert isometry_err(left) < ISO_TOL, label
    assert isometry_err(right.T) < ISO_TOL, label
    e_gpu = reconstruction_error(a, f)
    e_ref = float(np.linalg.norm(a - (U * S[None, :]) @ Vt))
    if e_ref > 1e-12 * np.linalg.norm(a):
        assert abs(e_gpu - e_ref) / e_ref < REC_TOL, (label, e_gpu, e_ref)
    else:
        assert e_gpu <= 1e-10 * np.linalg.norm(a), label
    j = _gapped_prefix(S, f.rank())
    if j:
        assert subspace_distance(left[:, :j], U[:, :j]) < SUB_TOL, label
        assert subspace_distance(right[:j].T, Vt[:j].T) < SUB_TOL, label
    if len(S) < f.rank() or True:
        assert f.discarded_weight == pytest.approx(dw, rel=1e-9, abs=1e-28), label


def test_golden_small_cases(cuda, golden_small):
    from paper_1710_01463_b200 import RsvdParams, rsvd

    names = sorted({k.split("/")[0] for k in golden_small.files})
    for name in names:
        a = golden_small[f"{name}/a"]
        k, ell, q, seed = (int(x) for x in golden_small[f"{name}/params"])
        f = rsvd(a, RsvdParams(k, ell, q, seed))
        ref = (golden_small[f"{name}/U"], golden_small[f"{name}/S"], golden_small[f"{name}/Vt"],
               float(golden_small[f"{name}/dw"][0]))
        check_against(a, f, ref, name)


def test_device_pointers_match_host_pointers(cuda, golden_small):
    import torch
    from paper_1710_01463_b200 import RsvdParams, rsvd

    a = golden_small["exp_200x160/a"]
    k, ell, q, seed = (int(x) for x in golden_small["exp_200x160/params"])
    fh = rsvd(a, RsvdParams(k, ell, q, seed))
    ad = torch.from_numpy(np.asfortranarray(a)).to(cuda)
    ad = ad.t().contiguous().t()
    fd = rsvd(ad, RsvdParams(k, ell, q, seed))
    assert np.array_equal(fh.sigma, fd.sigma.cpu().numpy())
    assert np.array_equal(fh.left, fd.left.cpu().numpy())
    assert np.array_equal(fh.right_adj, fd.right_adj.cpu().numpy())


def test_rsvd_matches_tsvd_fast_decay(cuda, oracle_mod, ref_mod):  # test_factorize.cpp:85-103
    from paper_1710_01463_b200 import RsvdParams, reconstruction_error, rsvd

    sigma = spectrum_family(0, 30)
    a = matrix_with_spectrum(oracle_mod, 3, 50, 30, sigma)
    Ut, St, Vtt, dwt = ref_mod.tsvd(a, 10)
    f = rsvd(a, RsvdParams(10, 20, 4, 123))
    assert f.rank() == 10 and not f.discarded_exact
    assert rel_sigma_err(f.sigma, St) < 1e-10
    et = float(np.linalg.norm(a - (Ut * St) @ Vtt))
    assert reconstruction_error(a, f) / et <= 1.01
    assert 0.0 < f.discarded_weight <= dwt * (1 + 1e-8)


@pytest.mark.parametrize("r", [3, 7])
def test_exact_rank_reconstructs(cuda, oracle_mod, r, ref_mod):  # test_factorize.cpp:105-120
    from paper_1710_01463_b200 import RsvdParams, reconstruction_error, rsvd

    sigma = [5.0 / (1.0 + k) for k in range(r)]
    a = matrix_with_spectrum(oracle_mod, 17 + r, 60, 40, sigma)
    f = rsvd(a, RsvdParams(10, 20, 4, 5))
    assert reconstruction_error(a, f) <= 1e-10 * np.linalg.norm(a)
    assert f.rank() <= 10
    ref = ref_mod.rsvd(a, 10, 20, 4, 5)
    assert f.rank() == len(ref[1])
    assert rel_sigma_err(f.sigma, ref[1]) < SIG_TOL


def test_zero_matrix(cuda):  # test_factorize.cpp:199-207
    from paper_1710_01463_b200 import RsvdParams, reconstruction_error, rsvd

    a = np.zeros((10, 6))
    f = rsvd(a, RsvdParams(3, 6, 2, 1))
    assert f.rank() == 0
    assert reconstruction_error(a, f) == 0.0


def test_deterministic_in_seed(cuda, oracle_mod):  # test_factorize.cpp:135-146
    from paper_1710_01463_b200 import RsvdParams, rsvd

    a = oracle_mod.gaussian_matrix(101, 48, 32)
    f1 = rsvd(a, RsvdParams(6, 12, 4, 77))
    f2 = rsvd(a, RsvdParams(6, 12, 4, 77))
    assert np.array_equal(f1.sigma, f2.sigma)
    assert np.array_equal(f1.left, f2.left)
    assert np.array_equal(f1.right_adj, f2.right_adj)
    f3 = rsvd(a, RsvdParams(6, 12, 4, 78))
    assert np.max(np.abs(f1.left - f3.left)) > 1e-12


def test_randomized_range_exact_rank(cuda, oracle_mod):  # test_factorize.cpp:163-173
    from paper_1710_01463_b200 import randomized_range

    a = matrix_with_spectrum(oracle_mod, 4, 30, 20, [4.0, 2.0, 1.0, 0.5, 0.25])
    q = randomized_range(a, 8, 2, 31)
    assert q.shape == (30, 8)
    assert isometry_err(q) < 1e-12
    assert np.linalg.norm(a - q @ (q.T @ a)) <= 1e-10 * np.linalg.norm(a)


def test_invalid_arguments(cuda):  # test_factorize.cpp:175-184
    from paper_1710_01463_b200 import InvalidArgument, RsvdParams, randomized_range, rsvd

    a = np.eye(4)
    with pytest.raises(InvalidArgument, match="rank must be >= 1"):
        rsvd(a, RsvdParams(0, 0, 4, 1))
    with pytest.raises(InvalidArgument, match="oversample must be >= rank"):
        rsvd(a, RsvdParams(3, 2, 4, 1))
    with pytest.raises(InvalidArgument, match="need 1 <= ell"):
        randomized_range(a, 0, 1, 1)
    with pytest.raises(InvalidArgument, match="need 1 <= ell"):
        randomized_range(a, 5, 1, 1)
    with pytest.raises(InvalidArgument, match="power must be >= 0"):
        randomized_range(a, 2, -1, 1)
    with pytest.raises(InvalidArgument, match="empty matrix"):
        rsvd(np.zeros((0, 3)), RsvdParams(1, 0, 1, 1))


def test_power_iterations_monotone(cuda, oracle_mod):  # test_factorize.cpp:209-226
    from paper_1710_01463_b200 import randomized_range

    sigma = 1.0 / np.arange(1, 25)
    mean = np.zeros(4)
    for trial in range(10):
        a = matrix_with_spectrum(oracle_mod, 1000 + trial, 40, 24, sigma)
        for i, q in enumerate([0, 1, 2, 4]):
            Q = randomized_range(a, 8, q, 7000 + trial)
            mean[i] += np.linalg.norm(a - Q @ (Q.T @ a)) / 10
    assert np.all(mean[1:] <= mean[:-1] * (1 + 1e-12))


def test_same_omega_as_oracle(cuda, oracle_mod, ref_mod):
    """Feeding the oracle the reference Omega vs its own gives the same
    answer to within the Omega ulp noise: parity is not an artefact of Omega."""
    from paper_1710_01463_b200 import RsvdParams, rsvd

    a = matrix_with_spectrum(oracle_mod, 77, 300, 250, np.exp(-np.arange(250) / 20.0))
    f = rsvd(a, RsvdParams(40, 50, 2, 4242))
    ref = ref_mod.rsvd(a, 40, 50, 2, 4242)
    check_against(a, f, ref, "omega")


def test_batched_matches_single(cuda, oracle_mod, ref_mod):
    import torch
    from paper_1710_01463_b200 import RsvdParams, rsvd, rsvd_batched

    m, n, bsz = 120, 90, 5
    mats = [matrix_with_spectrum(oracle_mod, 500 + b, m, n, 0.9 ** np.arange(90)) for b in
            range(bsz)]
    seeds = [1000 + b for b in range(bsz)]
    A = torch.from_numpy(np.stack([x.T for x in mats])).to(cuda).transpose(1, 2)
    bf = rsvd_batched(A, RsvdParams(20, 30, 2, 0), seeds)
    for b in range(bsz):
        ref = ref_mod.rsvd(mats[b], 20, 30, 2, seeds[b])
        fb = bf.item(b)
        fb.left, fb.sigma, fb.right_adj = (x.cpu().numpy() for x in (fb.left, fb.sigma,
                                                                    fb.right_adj))
        check_against(mats[b], fb, ref, f"batch{b}")
        single = rsvd(mats[b], RsvdParams(20, 30, 2, seeds[b]))
        assert rel_sigma_err(single.sigma, fb.sigma) < 1e-13


def test_host_pipelined_batch_equals_device(cuda, oracle_mod, monkeypatch):
    """Host-pointer batches are copied in chunks overlapped with compute; the
    factors must equal the device-pointer path item by item."""
    import torch
    from paper_1710_01463_b200 import RsvdParams, rsvd_batched

    monkeypatch.setenv("RSVD_HOST_CHUNKS", "3")
    m, n, bsz = 160, 128, 7
    mats = [matrix_with_spectrum(oracle_mod, 900 + b, m, n, 0.93 ** np.arange(n)) for b in
            range(bsz)]
    seeds = [77 + b for b in range(bsz)]
    host = torch.from_numpy(np.stack([x.T for x in mats])).transpose(1, 2).pin_memory()
    p = RsvdParams(12, 24, 2, 0)
    fh = rsvd_batched(host, p, seeds)
    fd = rsvd_batched(host.to(cuda), p, seeds)
    for b in range(bsz):
        r = fh.ranks[b]
        assert r == fd.ranks[b]
        assert rel_sigma_err(fh.sigma[b][:r].numpy(), fd.sigma[b][:r].cpu().numpy()) < 1e-13
        assert subspace_distance(fh.left[b][:, :r].numpy(), fd.left[b][:, :r].cpu().numpy()) < 1e-10


def _steep_or_mild(oracle_mod, b, m, n):
    """Even items: 2^-k spectrum (kappa(Y) >> tau^-1/2: the shifted-CholeskyQR
    fallback runs); odd items: mild 0.97^k (plain CholeskyQR2)."""
    sig = spectrum_family(0, min(m, n)) if b % 2 == 0 else 0.97 ** np.arange(min(m, n))
    return matrix_with_spectrum(oracle_mod, 4100 + b, m, n, sig)


def test_steep_spectrum_sampled_tail_matches_oracle(cuda, oracle_mod, ref_mod):
    """Sampled values far below sqrt(tau) sigma_0 (the pivot floor) must carry
    their true components like the reference's Householder bases: sigma and the
    discarded weight of a 2^-k spectrum against the oracle."""
    from paper_1710_01463_b200 import RsvdParams, rsvd

    a = matrix_with_spectrum(oracle_mod, 41, 200, 150, spectrum_family(0, 150))
    for k, ell, q in [(15, 40, 3), (10, 30, 0), (25, 50, 1)]:
        f = rsvd(a, RsvdParams(k, ell, q, 4040 + q))
        ref = ref_mod.rsvd(a, k, ell, q, 4040 + q)
        assert f.rank() == len(ref[1])
        # kept values above ~1e-6 sigma_0 are resolvable to 1e-10 by any
        # FP64 method; below that compare absolutely (u ||A|| scale)
        big = ref[1] > 1e-6 * ref[1][0]
        assert rel_sigma_err(f.sigma[big], ref[1][big]) < SIG_TOL
        assert np.max(np.abs(f.sigma - ref[1])) < 1e-14 * ref[1][0]
        assert f.discarded_weight == pytest.approx(ref[3], rel=1e-8, abs=1e-28)
        assert isometry_err(f.left) < ISO_TOL and isometry_err(f.right_adj.T) < ISO_TOL


def test_mixed_batch_fallback_masks(cuda, oracle_mod, ref_mod):
    """A batch mixing ill-conditioned and mild items: the masked fallback passes
    must touch only the ill items (every item against the oracle)."""
    import torch
    from paper_1710_01463_b200 import RsvdParams, rsvd_batched

    m, n, bsz = 256, 192, 6
    mats = [_steep_or_mild(oracle_mod, b, m, n) for b in range(bsz)]
    seeds = [300 + b for b in range(bsz)]
    A = torch.from_numpy(np.stack([x.T for x in mats])).to(cuda).transpose(1, 2)
    bf = rsvd_batched(A, RsvdParams(20, 48, 2, 0), seeds)
    for b in range(bsz):
        ref = ref_mod.rsvd(mats[b], 20, 48, 2, seeds[b])
        fb = bf.item(b)
        S = fb.sigma.cpu().numpy()
        assert fb.rank() == len(ref[1]), b
        big = ref[1] > 1e-6 * ref[1][0]
        assert rel_sigma_err(S[big], ref[1][big]) < SIG_TOL, b
        assert fb.discarded_weight == pytest.approx(ref[3], rel=1e-8, abs=1e-28), b
        assert isometry_err(fb.left.cpu().numpy()) < ISO_TOL, b


def test_rank_deficient_items_in_batch(cuda, oracle_mod, ref_mod):
    """Exact-rank items (Y rank deficient: the fallback plus basis completion)
    next to full-rank ones; the zero matrix too."""
    import torch
    from paper_1710_01463_b200 import RsvdParams, reconstruction_error, rsvd_batched

    m, n = 96, 80
    mats = [matrix_with_spectrum(oracle_mod, 70, m, n, [3.0, 2.0, 1.0]),
            matrix_with_spectrum(oracle_mod, 71, m, n, 0.9 ** np.arange(n)),
            np.zeros((m, n)),
            matrix_with_spectrum(oracle_mod, 72, m, n, [5.0] * 7)]
    seeds = [5, 6, 7, 8]
    A = torch.from_numpy(np.stack([x.T for x in mats])).to(cuda).transpose(1, 2)
    bf = rsvd_batched(A, RsvdParams(10, 20, 2, 0), seeds)
    for b, a in enumerate(mats):
        ref = ref_mod.rsvd(a, 10, 20, 2, seeds[b])
        fb = bf.item(b)
        fb.left, fb.sigma, fb.right_adj = (x.cpu().numpy() for x in (fb.left, fb.sigma,
                                                                    fb.right_adj))
        assert fb.rank() == len(ref[1]), b
        if fb.rank():
            assert rel_sigma_err(fb.sigma, ref[1]) < SIG_TOL, b
            assert isometry_err(fb.left) < ISO_TOL, b
        if b != 1:
            assert reconstruction_error(a, fb) <= 1e-10 * max(np.linalg.norm(a), 1.0), b


def test_batched_out_buffers_reused(cuda, oracle_mod):
    """rsvd_batched(..., out=prev) writes into the previous result's buffers
    (pinned host factors reused in a loop) with identical values."""
    import torch
    from paper_1710_01463_b200 import InvalidArgument, RsvdParams, rsvd_batched

    m, n, bsz = 96, 80, 4
    mats = [matrix_with_spectrum(oracle_mod, 600 + b, m, n, 0.9 ** np.arange(n)) for b in range(bsz)]
    seeds = [11 + b for b in range(bsz)]
    host = torch.from_numpy(np.stack([x.T for x in mats])).transpose(1, 2).pin_memory()
    p = RsvdParams(10, 20, 2, 0)
    first = rsvd_batched(host, p, seeds)
    ptr = first.left.data_ptr()
    again = rsvd_batched(host, p, seeds, out=first)
    assert again.left.data_ptr() == ptr
    ref = rsvd_batched(host, p, seeds)
    assert torch.equal(again.sigma, ref.sigma) and torch.equal(again.left, ref.left)
    dev = rsvd_batched(host.to(cuda), p, seeds)
    dev2 = rsvd_batched(host.to(cuda), p, seeds, out=dev)
    assert torch.equal(dev2.sigma.cpu(), ref.sigma)
    with pytest.raises(InvalidArgument, match="out= buffers"):
        rsvd_batched(host[:2], p, seeds[:2], out=first)


_NO_GRAPH_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1710_01463_b200 import RsvdParams, rsvd_batched
rng = np.random.default_rng(5)
a = torch.from_numpy(rng.standard_normal((6, 96, 80))).to("cuda:0").transpose(1, 2)
p = RsvdParams(10, 20, 2, 0)
for _ in range(3):  # the graph path captures on the second call and replays on the third
    f = rsvd_batched(a, p, list(range(6)))
torch.cuda.synchronize()
np.save({out!r}, np.concatenate([f.sigma.cpu().numpy().ravel(), f.left.cpu().numpy().ravel()]))
"""


def test_graph_replay_equals_direct_launches(cuda, tmp_path):
    """RSVD_NO_GRAPH=1 (direct launches, no CUDA-graph capture) gives bitwise
    the same factors as the captured-and-replayed path."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_graph in ("0", "1"):
        out = str(tmp_path / f"f{env_graph}.npy")
        env = dict(os.environ)
        env.pop("RSVD_NO_GRAPH", None)
        if env_graph == "1":
            env["RSVD_NO_GRAPH"] = "1"
        subprocess.run([sys.executable, "-c", _NO_GRAPH_SCRIPT.format(root=root, out=out)],
                       check=True, env=env, timeout=300)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


_GEMM_PATH_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth
cfg = synth.CONFIGS["C4"]
A = synth.make_batch(cfg, device="cuda:0")[:8].contiguous()
seeds = synth.omega_seeds(cfg)[:8]
f = rsvd_batched(A, RsvdParams(cfg.rank, cfg.ell, cfg.power, 0), seeds)
torch.cuda.synchronize()
r = min(f.ranks)
np.savez({out!r}, s=f.sigma[:, :r].cpu().numpy(), u=f.left[:, :, :r].cpu().numpy(),
         dw=np.array(f.discarded_weight))
"""


def test_ozaki_and_dmma_a_passes_agree(cuda, tmp_path):
    """The emulated-FP64 A-passes (INT8 tensor cores, the default for C4-sized
    batches) and RSVD_FP64_GEMM=dmma give the same factorization of 8 C4 items
    to the north_star tolerances (sigma 1e-10 relative, U to 1e-8 in subspace
    distance on the gapped prefix, discarded weight 1e-8)."""
    import os
    import subprocess
    import sys

    from tests.helpers import subspace_distance

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for path in ("ozaki", "dmma"):
        out = str(tmp_path / f"{path}.npz")
        env = dict(os.environ)
        env.pop("RSVD_FP64_GEMM", None)
        if path == "dmma":
            env["RSVD_FP64_GEMM"] = "dmma"
        subprocess.run([sys.executable, "-c", _GEMM_PATH_SCRIPT.format(root=root, out=out)],
                       check=True, env=env, timeout=600)
        res[path] = np.load(out)
    s0, s1 = res["ozaki"]["s"], res["dmma"]["s"]
    assert np.max(np.abs(s0 - s1) / s1[:, :1]) < 1e-12
    assert np.max(np.abs(s0 - s1) / s1) < 1e-10
    for b in range(s0.shape[0]):
        assert subspace_distance(res["ozaki"]["u"][b, :, :200], res["dmma"]["u"][b, :, :200]) < 1e-8
    assert np.allclose(res["ozaki"]["dw"], res["dmma"]["dw"], rtol=1e-8, atol=0)
