"""Host-side pieces of the TEBD bond update (no GPU): models and gates
(restating test_models.cpp), the random product state (test_mps.cpp:82-108,
against the oracle), layer validation."""
import numpy as np
import pytest

from tests import tebd_helpers as TH
from tests import tebd_models as M
from paper_1710_01463_b200._lib import InvalidArgument

from .tebd_helpers import mps_to_dense


def test_spin_half_and_one():  # test_models.cpp:48-70
    a = M.spin_operators(0.5)
    assert a.dim == 2
    assert np.array_equal(a.x, [[0, 0.5], [0.5, 0]])
    assert np.array_equal(a.z, [[-0.5, 0], [0, 0.5]])
    assert np.array_equal(a.parity, [[1, 0], [0, -1]])
    b = M.spin_operators(1.0)
    r = 1.0 / np.sqrt(2.0)
    assert np.max(np.abs(b.x - [[0, r, 0], [r, 0, r], [0, r, 0]])) < 1e-15
    assert list(np.diag(b.parity)) == [1, -1, 1]


@pytest.mark.parametrize("s", [0.5, 1.0, 1.5, 2.0, 5.0])
def test_spin_algebra_identities(s):  # test_models.cpp:71-86
    a = M.spin_operators(s)
    x, z = a.x.astype(complex), a.z.astype(complex)
    y = -1j * (z @ x - x @ z)
    cas = x @ x + y @ y + z @ z
    assert np.max(np.abs(cas - s * (s + 1) * np.eye(a.dim))) < 1e-12
    assert np.max(np.abs(x @ y - y @ x - 1j * z)) < 1e-12
    assert np.max(np.abs(a.parity @ a.x + a.x @ a.parity)) < 1e-15


def test_invalid_spins():  # test_models.cpp:88-92
    for s in (0.0, 0.3, -1.0):
        with pytest.raises(InvalidArgument):
            M.spin_operators(s)


def test_parity_structures():  # test_models.cpp:94-117
    st = M.parity_structure(M.ChainModel(4, 5.0, 1.0))
    assert (st.dim, st.dim_even, st.dim_odd) == (11, 6, 5)
    assert st.charges == [k % 2 for k in range(11)]
    s2 = M.parity_structure(M.CylinderModel(4, 2, 3.0))
    assert (s2.dim, s2.dim_even, s2.dim_odd, s2.charges) == (4, 2, 2, [0, 1, 1, 0])
    s3 = M.parity_structure(M.CylinderModel(4, 3, 3.0))
    assert (s3.dim, s3.dim_even, s3.dim_odd) == (8, 4, 4)


def _dense_chain(spin, length, field):
    a = M.spin_operators(spin)
    d = a.dim

    def at(op, j):
        out = np.eye(1)
        for k in range(length):
            out = np.kron(out, op if k == j else np.eye(d))
        return out

    h = sum(-(1 / spin ** 2) * at(a.x, j) @ at(a.x, j + 1) for j in range(length - 1))
    return h + sum((field / spin) * at(a.z, j) for j in range(length))


def _from_bonds(model):
    bonds = M.bond_hamiltonians(model)
    d = int(round(np.sqrt(bonds[0].shape[0])))
    n = model.length
    h = np.zeros((d ** n, d ** n))
    for b, hb in enumerate(bonds):
        h += np.kron(np.kron(np.eye(d ** b), hb), np.eye(d ** (n - b - 2)))
    return h


@pytest.mark.parametrize("spin,length", [(0.5, 2), (0.5, 5), (1.0, 3), (2.5, 3)])
def test_bond_terms_sum_to_chain_hamiltonian(spin, length):  # test_models.cpp:119-128
    direct = _dense_chain(spin, length, 1.3)
    fb = _from_bonds(M.ChainModel(length, spin, 1.3))
    assert np.max(np.abs(direct - fb)) < 1e-12 * np.max(np.abs(direct))


def test_bond_terms_conserve_parity_and_are_symmetric():  # test_models.cpp:140-148
    for m in (M.ChainModel(4, 1.0, 0.7), M.CylinderModel(3, 2, 3.0)):
        st = M.parity_structure(m)
        for h in M.bond_hamiltonians(m):
            assert np.array_equal(h, h.T)
            assert M._commutes_with_parity(h, st.charges)
    with pytest.raises(InvalidArgument, match="at least two sites"):
        M.bond_hamiltonians(M.ChainModel(1, 0.5, 1.0))
    with pytest.raises(InvalidArgument, match="width must be >= 2"):
        M.parity_structure(M.CylinderModel(3, 1, 1.0))


def _series_exp(a):
    out = np.eye(a.shape[0])
    term = np.eye(a.shape[0])
    for k in range(1, 60):
        term = term @ a / k
        out = out + term
    return out


def test_gates():  # test_models.cpp:193-250
    st = M.parity_structure(M.ChainModel(2, 0.5, 1.0))
    g = M.build_gate(M.bond_hamiltonians(M.ChainModel(2, 0.5, 1.0))[0], st.charges, 0.0)
    assert np.max(np.abs(g.block - np.eye(4))) < 1e-14
    for m in (M.ChainModel(3, 1.0, 0.9), M.CylinderModel(3, 2, 3.1)):
        st = M.parity_structure(m)
        h = M.bond_hamiltonians(m)[0]
        for dt in (0.05, 0.4):
            g = M.build_gate(h, st.charges, dt)
            ref = _series_exp(-dt * h)
            assert np.max(np.abs(g.block - ref)) < 1e-12 * np.max(np.abs(ref))
    sx = np.array([[0.0, 1.0], [1.0, 0.0]])
    g = M.build_gate(-np.kron(sx, sx), [0, 1], 0.3, M.GateForm.product)
    assert len(g.terms) == 2 and g.terms[0].weight >= g.terms[1].weight
    assert np.max(np.abs(sum(np.kron(t.left, t.right) for t in g.terms) - g.block)) < 1e-12
    for m in (M.ChainModel(3, 1.5, 1.2), M.CylinderModel(3, 2, 2.8)):
        st = M.parity_structure(m)
        g = M.build_gate(M.bond_hamiltonians(m)[0], st.charges, 0.25, M.GateForm.product)
        d = st.dim
        total = np.zeros((d * d, d * d))
        for t in g.terms:
            total += np.kron(t.left, t.right)
            for r in range(d):
                for c in range(d):
                    if (st.charges[r] ^ st.charges[c]) != t.charge:
                        assert t.left[r, c] == 0.0 and t.right[r, c] == 0.0
        assert np.max(np.abs(total - g.block)) < 1e-12
        assert all(g.terms[k].weight >= g.terms[k + 1].weight for k in range(len(g.terms) - 1))


def test_gate_validation():  # test_models.cpp:252-272
    sx = np.array([[0.0, 1.0], [1.0, 0.0]])
    sz = np.array([[-1.0, 0.0], [0.0, 1.0]])
    good = -np.kron(sx, sx) + np.kron(sz, np.eye(2))
    for args in ((good, [0, 1], -0.1), (np.eye(3), [0, 1], 0.1),
                 (np.kron(sx, np.eye(2)), [0, 1], 0.1)):
        with pytest.raises(InvalidArgument):
            M.build_gate(*args)
    for tol in (0.0, 1.0):
        with pytest.raises(InvalidArgument):
            M.build_gate(good, [0, 1], 0.1, M.GateForm.block, tol)
    asym = good.copy()
    asym[0, 3] += 0.5
    with pytest.raises(InvalidArgument, match="symmetric"):
        M.build_gate(asym, [0, 1], 0.1)


@pytest.mark.parametrize("seed", [1, 2, 99])
def test_random_product_state_matches_oracle(seed):  # test_mps.cpp:82-108
    from oracle import tebd_oracle

    from paper_1710_01463_b200 import tebd

    st = M.parity_structure(M.ChainModel(6, 1.0, 1.0))
    psi = TH.random_product_state(st, 6, seed, device="cpu")
    psi.validate()
    assert psi.max_bond_dimension() == 1
    g, lam = psi.to_numpy()
    go, lo = tebd_oracle.random_product_state(st.charges, 6, seed)
    v = mps_to_dense(g, lam, st.charges)
    assert np.array_equal(v, mps_to_dense(go, lo, st.charges))
    assert abs(np.linalg.norm(v) - 1.0) < 1e-14
    # global parity even: the single nonzero basis state has even total charge
    idx = int(np.flatnonzero(v)[0])
    q = 0
    for _ in range(6):
        q ^= st.charges[idx % st.dim]
        idx //= st.dim
    assert q == 0


def test_product_state_deterministic_in_seed():  # test_mps.cpp:96-108
    from paper_1710_01463_b200 import tebd

    st = M.parity_structure(M.CylinderModel(5, 2, 3.0))
    a = mps_to_dense(*TH.random_product_state(st, 5, 7, device="cpu").to_numpy(), st.charges)
    b = mps_to_dense(*TH.random_product_state(st, 5, 7, device="cpu").to_numpy(), st.charges)
    assert np.array_equal(a, b)
    assert any(not np.array_equal(
        mps_to_dense(*TH.random_product_state(st, 5, s, device="cpu").to_numpy(), st.charges), a)
        for s in range(8, 16))


def test_validate_rejects_corrupted_states():  # test_mps.cpp:475-492
    import torch

    from paper_1710_01463_b200 import tebd

    st = M.parity_structure(M.ChainModel(4, 0.5, 1.0))
    psi = TH.random_product_state(st, 4, 3, device="cpu")
    psi.gammas[1][0][0] = torch.zeros(3, 3, dtype=torch.float64)
    with pytest.raises(ValueError, match="fusion rule"):
        psi.validate()
    psi = TH.random_product_state(st, 4, 3, device="cpu")
    psi.lambdas.pop()
    with pytest.raises(ValueError, match="one bond more"):
        psi.validate()
