"""GPU TEBD bond update against dense evolution and the
oracle's restatement of apply_gate (mps.cpp:111-323).  Restates
test_mps.cpp:110-216 (identity gate, dense evolution on chain and cylinder,
block vs product forms, truncation tail, lambdas = Schmidt values) plus
oracle parity and layer batching.  Singular-vector signs are a gauge freedom,
so comparisons use gauge-invariant quantities: Schmidt values, discarded
weights, the dense state."""
import numpy as np
import pytest

from tests import tebd_helpers as TH
from tests import tebd_models as M

from .tebd_helpers import apply_two_site, mps_to_dense, schmidt_values, sorted_lambdas

pytestmark = pytest.mark.gpu


def _req(chi, maximal=True):
    from paper_1710_01463_b200 import RankPolicy, SectorRankRequest

    return SectorRankRequest(RankPolicy.maximal if maximal else RankPolicy.per_sector_estimate,
                             chi)


def _to_device(site, g, lam, cuda):
    import torch

    from paper_1710_01463_b200 import tebd

    gd = [[[torch.from_numpy(np.ascontiguousarray(x)).to(cuda) for x in pair] for pair in s]
          for s in g]
    ld = [[torch.from_numpy(np.ascontiguousarray(x)).to(cuda) for x in pair] for pair in lam]
    return tebd.SymmetricMPS(site, gd, ld)


def _entangled(model, chi, dt, passes, seed, cuda):
    """Oracle-built entangled state (random product state + `passes` layers of
    block gates, exact factorization), moved to the device."""
    from oracle import tebd_oracle

    st = M.parity_structure(model)
    n = model.length
    g, lam = tebd_oracle.random_product_state(st.charges, n, seed)
    bonds = M.bond_hamiltonians(model)
    for ps in range(passes):
        for b in range(ps % 2, n - 1, 2):
            gate = M.build_gate(bonds[b], st.charges, dt)
            tebd_oracle.apply_gate(g, lam, st.charges, b, gate.block, None, "block", chi,
                                   maximal=True)
    tebd_oracle.canonicalize(g, lam, st.charges)  # helpers.hpp entangled_state ends canonical
    return st, g, lam, _to_device(st, g, lam, cuda)


def test_identity_gate_leaves_state_invariant(cuda):  # test_mps.cpp:110-126
    from paper_1710_01463_b200 import BlockMethod, tebd

    m = M.ChainModel(5, 0.5, 1.0)
    st, g, lam, psi = _entangled(m, 16, 0.3, 2, 3, cuda)
    before = mps_to_dense(g, lam, st.charges)
    bonds = M.bond_hamiltonians(m)
    for b in range(4):
        gate = M.build_gate(bonds[b], st.charges, 0.0)
        tebd.apply_gate(psi, b, gate, 64, BlockMethod.deterministic(), _req(64))
    after = mps_to_dense(*psi.to_numpy(), st.charges)
    assert np.linalg.norm(before - after) < 1e-11


@pytest.mark.parametrize("model,seed", [(M.ChainModel(4, 0.5, 1.0), 11),
                                        (M.ChainModel(3, 1.0, 1.4), 5),
                                        (M.CylinderModel(3, 2, 3.0), 21)])
def test_matches_dense_evolution(cuda, model, seed):  # test_mps.cpp:42-79, 128-137
    from paper_1710_01463_b200 import BlockMethod, tebd

    st = M.parity_structure(model)
    n = model.length
    psi = TH.random_product_state(st, n, seed, device=cuda)
    ref = mps_to_dense(*psi.to_numpy(), st.charges)
    bonds = M.bond_hamiltonians(model)
    dts = [0.2, 0.35, 0.1]
    gi = 0
    for ps in range(3):
        for b in range(ps % 2, n - 1, 2):
            gate = M.build_gate(bonds[b], st.charges, dts[gi % 3])
            gi += 1
            tebd.apply_gate(psi, b, gate, 256, BlockMethod.deterministic(), _req(256))
            ref = apply_two_site(ref, gate.block, b, n, st.dim)
            ref /= np.linalg.norm(ref)
            got = mps_to_dense(*psi.to_numpy(), st.charges)
            assert abs(ref @ got) / np.linalg.norm(got) == pytest.approx(1.0, abs=1e-10)
            assert np.linalg.norm(got) == pytest.approx(1.0, rel=2e-2)
    psi.validate()


@pytest.mark.parametrize("model,seed,form", [(M.ChainModel(4, 0.5, 1.0), 11, "block"),
                                             (M.CylinderModel(3, 2, 3.0), 21, "block"),
                                             (M.ChainModel(4, 0.5, 1.0), 7, "product")])
def test_complex_mps_matches_dense_evolution(cuda, model, seed, form):
    """check_against_dense_evolution<Complex> (test_mps.cpp:128-137): a
    SymmetricMPS<Complex> evolved by the same real gates; every bond update runs
    the complex factorization (complex Gammas, arbitrary singular-vector
    phases), the state must track the dense evolution."""
    import torch

    from paper_1710_01463_b200 import BlockMethod, tebd

    st = M.parity_structure(model)
    n = model.length
    psi = TH.random_product_state(st, n, seed, device=cuda, dtype=torch.complex128)
    ref = mps_to_dense(*psi.to_numpy(), st.charges)
    assert np.iscomplexobj(ref)
    bonds = M.bond_hamiltonians(model)
    gf = M.GateForm.block if form == "block" else M.GateForm.product
    dts = [0.2, 0.35, 0.1]
    gi = 0
    for ps in range(3):
        for b in range(ps % 2, n - 1, 2):
            gate = M.build_gate(bonds[b], st.charges, dts[gi % 3], gf)
            gi += 1
            meth = BlockMethod.deterministic() if gi % 2 else BlockMethod.randomized(4, 99)
            tebd.apply_gate(psi, b, gate, 256, meth, _req(256))
            ref = apply_two_site(ref, gate.block, b, n, st.dim)
            ref /= np.linalg.norm(ref)
            got = mps_to_dense(*psi.to_numpy(), st.charges)
            assert abs(np.vdot(ref, got)) / np.linalg.norm(got) == pytest.approx(1.0, abs=1e-10)
    assert psi.gammas[0][0][0].dtype == torch.complex128
    psi.validate()
    TH.canonicalize(psi)
    assert TH.lambda_norm_error(psi) < 1e-12


def test_block_and_product_forms_agree(cuda):  # test_mps.cpp:139-161
    from paper_1710_01463_b200 import BlockMethod, tebd

    for m in (M.ChainModel(4, 1.0, 1.1), M.CylinderModel(3, 2, 2.9)):
        st = M.parity_structure(m)
        n = m.length
        pb = TH.random_product_state(st, n, 31, device=cuda)
        pp = TH.random_product_state(st, n, 31, device=cuda)
        bonds = M.bond_hamiltonians(m)
        for ps in range(2):
            for b in range(ps, n - 1, 2):
                h = bonds[b]
                tebd.apply_gate(pb, b, M.build_gate(h, st.charges, 0.25, M.GateForm.block), 256,
                                BlockMethod.deterministic(), _req(256))
                tebd.apply_gate(pp, b, M.build_gate(h, st.charges, 0.25, M.GateForm.product),
                                256, BlockMethod.deterministic(), _req(256))
        vb = mps_to_dense(*pb.to_numpy(), st.charges)
        vp = mps_to_dense(*pp.to_numpy(), st.charges)
        assert abs(vb @ vp) == pytest.approx(1.0, abs=1e-10)


def test_truncation_reports_dense_schmidt_tail(cuda):  # test_mps.cpp:163-196
    from paper_1710_01463_b200 import BlockMethod, tebd

    m = M.ChainModel(4, 0.5, 1.0)
    st, g, lam, psi = _entangled(m, 64, 0.4, 2, 17, cuda)
    ref = mps_to_dense(g, lam, st.charges)
    bond = 1
    gate = M.build_gate(M.bond_hamiltonians(m)[bond], st.charges, 0.5)
    ref = apply_two_site(ref, gate.block, bond, 4, st.dim)
    sch = schmidt_values(ref, bond + 1, 4, st.dim)
    chi = 2
    stats = tebd.apply_gate(psi, bond, gate, chi, BlockMethod.deterministic(), _req(chi))
    total = float(np.sum(sch ** 2))
    kept = float(np.sum(sch[:chi] ** 2))
    assert stats.discarded_weight == pytest.approx((total - kept) / total, rel=1e-9)
    assert stats.mid_rank == chi and psi.bond_dimension(bond + 1) == chi
    ks = schmidt_values(mps_to_dense(*psi.to_numpy(), st.charges), bond + 1, 4, st.dim)
    np.testing.assert_allclose(ks[:chi], sch[:chi] / np.sqrt(kept), rtol=1e-9)


def test_lambdas_are_schmidt_values(cuda):  # test_mps.cpp:198-215 (GPU-evolved state)
    from paper_1710_01463_b200 import BlockMethod, tebd

    for m in (M.ChainModel(5, 0.5, 0.9), M.CylinderModel(3, 2, 3.1)):
        st = M.parity_structure(m)
        n = m.length
        psi = TH.random_product_state(st, n, 23, device=cuda)
        bonds = M.bond_hamiltonians(m)
        for ps in range(3):
            for b in range(ps % 2, n - 1, 2):
                tebd.apply_gate(psi, b, M.build_gate(bonds[b], st.charges, 0.35), 64,
                                BlockMethod.deterministic(), _req(64))
        TH.canonicalize(psi)  # mps.cpp:326-350
        assert TH.lambda_norm_error(psi) < 1e-12
        v = mps_to_dense(*psi.to_numpy(), st.charges)
        assert np.linalg.norm(v) == pytest.approx(1.0, abs=1e-10)
        for b in range(1, n):
            dense = schmidt_values(v, b, n, st.dim)
            lam = sorted_lambdas(psi.lambdas[b])
            np.testing.assert_allclose(lam, dense[:len(lam)], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("form", ["block", "product"])
@pytest.mark.parametrize("kind", ["tsvd", "rsvd"])
def test_apply_gate_vs_oracle(cuda, form, kind):
    """A larger chain (spin 1, L = 8) evolved by GPU and oracle side by side:
    per-sector Schmidt values (1e-10), discarded weights and the dense state."""
    from oracle import tebd_oracle

    from paper_1710_01463_b200 import BlockMethod, tebd

    m = M.ChainModel(8, 1.0, 1.2)
    st, g, lam, psi = _entangled(m, 40, 0.3, 4, 41, cuda)
    bonds = M.bond_hamiltonians(m)
    gf = M.GateForm.block if form == "block" else M.GateForm.product
    meth = BlockMethod.randomized(4, 77) if kind == "rsvd" else BlockMethod.deterministic()
    meth.rsvd_min_dim = 8
    chi = 24
    for ps in range(2):
        for b in range(ps % 2, m.length - 1, 2):
            gate = M.build_gate(bonds[b], st.charges, 0.2, gf)
            stats = tebd.apply_gate(psi, b, gate, chi, meth, _req(chi, maximal=False))
            terms = [(t.left, t.right, t.charge) for t in gate.terms]
            dw, rank, _ = tebd_oracle.apply_gate(g, lam, st.charges, b, gate.block, terms, form,
                                                 chi, kind=kind, power=4, seed=77, min_dim=8)
            assert stats.mid_rank == rank, b
            assert stats.discarded_weight == pytest.approx(dw, rel=1e-8, abs=1e-15), b
            for s in (0, 1):
                got = psi.lambdas[b + 1][s].cpu().numpy()
                # values are normalised (sum lambda^2 = 1): 1e-10 relative above
                # 1e-4, otherwise the O(u)-level absolute gauge noise of two
                # independent evolutions (~1e-13 after a few gates)
                np.testing.assert_allclose(got, lam[b + 1][s], rtol=1e-10, atol=1e-12)
    v_gpu = mps_to_dense(*psi.to_numpy(), st.charges)
    v_ref = mps_to_dense(g, lam, st.charges)
    assert abs(v_gpu @ v_ref) / (np.linalg.norm(v_gpu) * np.linalg.norm(v_ref)) == \
        pytest.approx(1.0, abs=1e-9)


def test_layer_equals_sequential(cuda):
    """apply_gate_layer (one batched factorization for the whole layer) gives
    the same state as gate-by-gate application."""
    from paper_1710_01463_b200 import BlockMethod, tebd

    m = M.ChainModel(10, 0.5, 1.0)
    st, g, lam, psi_a = _entangled(m, 32, 0.3, 3, 5, cuda)
    psi_b = _to_device(st, g, lam, cuda)
    bonds = M.bond_hamiltonians(m)
    for meth in (BlockMethod.deterministic(), BlockMethod.randomized(3, 9)):
        meth.rsvd_min_dim = 4
        for ps in range(2):
            layer = list(range(ps % 2, m.length - 1, 2))
            gates = [M.build_gate(bonds[b], st.charges, 0.25) for b in layer]
            sa = tebd.apply_gate_layer(psi_a, layer, gates, 16, meth, _req(16, maximal=False))
            sb = [tebd.apply_gate(psi_b, b, gt, 16, meth, _req(16, maximal=False))
                  for b, gt in zip(layer, gates)]
            for x, y in zip(sa, sb):
                assert x.mid_rank == y.mid_rank
                assert x.discarded_weight == pytest.approx(y.discarded_weight, rel=1e-9,
                                                           abs=1e-14)
    va = mps_to_dense(*psi_a.to_numpy(), st.charges)
    vb = mps_to_dense(*psi_b.to_numpy(), st.charges)
    assert abs(va @ vb) / (np.linalg.norm(va) * np.linalg.norm(vb)) == pytest.approx(1.0, abs=1e-9)
    with pytest.raises(Exception, match="disjoint"):
        tebd.apply_gate_layer(psi_a, [0, 1], [gates[0], gates[0]], 16, meth)
