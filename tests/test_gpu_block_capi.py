"""rsvd_block_factorize_f64 -- block_factorize (blocks.cpp:38-118) behind the
C ABI for C++ callers -- against the reference's own block_factorize
(oracle/_ref, proj/src/blocks.cpp compiled unmodified), with host and device
buffers: kept ranks, singular values, discarded weights, the exact flag and
the reference's error messages."""
import ctypes

import numpy as np
import pytest

from tests.helpers import isometry_err

pytestmark = pytest.mark.gpu


def capi_block_factorize(blocks, charges, chi, maximal=False, slack=-1, kind="tsvd",
                         oversample=0, power=4, seed=0, min_dim=32, device=False):
    import torch

    from paper_1710_01463_b200 import _lib as L

    h = L.default_handle()
    ns = len(blocks)
    bl = [np.asfortranarray(b, dtype=np.float64) for b in blocks]
    rows = np.array([b.shape[0] for b in bl], dtype=np.int64)
    cols = np.array([b.shape[1] for b in bl], dtype=np.int64)
    cap = [max(1, min(r, c, chi)) for r, c in zip(rows, cols)]
    keep = []

    def buf(shape):
        if device:
            t = torch.zeros(shape[::-1], dtype=torch.float64, device="cuda:0").t()
            keep.append(t)
            return t, t.data_ptr()
        a = np.zeros(shape, order="F")
        keep.append(a)
        return a, a.ctypes.data

    ins, ptrs = [], []
    for b in bl:
        if device:
            t = torch.from_numpy(np.ascontiguousarray(b.T)).to("cuda:0").t() if b.size else \
                torch.zeros(b.shape[::-1], dtype=torch.float64, device="cuda:0").t()
            ins.append(t)
            ptrs.append(t.data_ptr() if b.size else 0)
        else:
            ins.append(b)
            ptrs.append(b.ctypes.data if b.size else 0)
    U = [buf((max(int(r), 1), k)) for r, k in zip(rows, cap)]
    S = [buf((k, 1)) for k in cap]
    V = [buf((k, max(int(c), 1))) for k, c in zip(cap, cols)]
    P = ctypes.c_void_p * ns
    ld = np.maximum(rows, 1)
    ldu = np.maximum(rows, 1)
    ldvt = np.array(cap, dtype=np.int64)
    ch = np.asarray(charges, dtype=np.int64)
    out_rank = np.zeros(ns, dtype=np.int64)
    sdw = np.zeros(ns)
    tot = ctypes.c_double(0.0)
    ex = ctypes.c_int(0)
    rc = L.load().rsvd_block_factorize_f64(
        h.raw, ns, ch.ctypes.data, P(*ptrs), rows.ctypes.data, cols.ctypes.data, ld.ctypes.data,
        chi, int(maximal), slack, 1 if kind == "rsvd" else 0, oversample, power, seed, min_dim,
        P(*[u[1] for u in U]), ldu.ctypes.data, P(*[s[1] for s in S]), P(*[v[1] for v in V]),
        ldvt.ctypes.data, out_rank.ctypes.data, sdw.ctypes.data, ctypes.byref(tot),
        ctypes.byref(ex), L.PTR_DEVICE if device else L.PTR_HOST)
    L.raise_for(rc, h.raw)
    out = []
    for s in range(ns):
        r = int(out_rank[s])

        def host(x):
            return x.cpu().numpy() if device else x

        out.append((host(U[s][0])[:rows[s], :r], host(S[s][0])[:r, 0],
                    host(V[s][0])[:r, :cols[s]], float(sdw[s])))
    return out, tot.value, bool(ex.value)


def _sectors(seed, shapes, decay=6.0):
    rng = np.random.default_rng(seed)
    return [np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / decay)[None, :])
            for (m, n) in shapes]


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("kind,shapes,charges,chi,over,maximal", [
    ("rsvd", [(40, 36), (48, 40)], [0, 1], 16, 0, False),
    ("rsvd", [(64, 40), (20, 30), (33, 50), (64, 40)], [3, 0, 1, 7], 24, 20, False),
    ("tsvd", [(12, 9), (7, 15)], [1, 0], 10, 0, True),
    ("rsvd", [(36, 36), (36, 36)], [5, 2], 40, 500, False),
    ("rsvd", [(40, 40), (0, 5)], [0, 1], 8, 4, False),
])
def test_block_factorize_capi_matches_reference(cuda, ref_mod, device, kind, shapes, charges,
                                                chi, over, maximal):
    bl = _sectors(sum(charges) + chi, shapes)
    got, tot, ex = capi_block_factorize(bl, charges, chi, maximal=maximal, kind=kind,
                                        oversample=over, power=2, seed=99, device=device)
    ref, rtot, rex = ref_mod.block_factorize(bl, charges, chi, maximal=maximal, kind=kind,
                                             oversample=over, power=2, seed=99)
    assert ex == rex
    assert tot == pytest.approx(rtot, rel=1e-8, abs=1e-24)
    for s, ((U, S, Vt, dw), (Ur, Sr, Vtr, dwr)) in enumerate(zip(got, ref)):
        assert len(S) == len(Sr), s
        if len(S):
            assert np.max(np.abs(S - Sr) / Sr) < 1e-10, s
            assert isometry_err(U) < 1e-12 and isometry_err(Vt.T) < 1e-12
            a = bl[s]
            assert np.linalg.norm(a - (U * S) @ Vt) == pytest.approx(
                np.linalg.norm(a - (Ur * Sr) @ Vtr), rel=1e-9, abs=1e-13)
        assert dw == pytest.approx(dwr, rel=1e-8, abs=1e-24), s


def test_block_factorize_capi_ties_and_errors(cuda, ref_mod):
    """Exact ties go to the lower charge (test_blocks.cpp:114-140); argument
    errors carry the reference's messages."""
    from paper_1710_01463_b200 import InvalidArgument

    bl = [np.diag([2.0, 1.0]), np.diag([2.0, 1.0])]
    got, _, _ = capi_block_factorize(bl, [7, 3], 3, maximal=True)
    ref, _, _ = ref_mod.block_factorize(bl, [7, 3], 3, maximal=True)
    assert [len(g[1]) for g in got] == [len(r[1]) for r in ref] == [1, 2]
    a = np.eye(3)
    for blocks, ch, chi in (([a, a], [0, 0], 2), ([a], [0], 0)):
        with pytest.raises(InvalidArgument) as eg:
            capi_block_factorize(blocks, ch, chi)
        with pytest.raises(ref_mod.RefInvalid) as er:
            ref_mod.block_factorize(blocks, ch, chi)
        assert str(eg.value) == str(er.value)
