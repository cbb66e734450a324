"""TEST INFRASTRUCTURE: model and gate construction feeding the TEBD
bond-update tests and tools/tebd_bench.py (model construction is out of the
hot-path scope; the product keeps only the gate / site
interface types, paper_1710_01463_b200/gates.py).

Restates rlftn's models.hpp / models.cpp: spin operators (models.cpp:121-145),
the Z2 parity structure (models.cpp:151-158), the two-site bond Hamiltonians of
the transverse-field chain and cylinder (models.cpp:160-178) and
`build_gate` (models.cpp:180-247: exp(-dt h) by symmetric eigensolver and, for
GateForm.product, the per-pair-charge operator Schmidt decomposition).  These
are d^2 x d^2 setup computations done once per time step; they feed the GPU
bond update in tebd.py.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List, Union

import numpy as np

from paper_1710_01463_b200._lib import InvalidArgument
from paper_1710_01463_b200.gates import GateForm, KronTerm, SiteStructure, TwoSiteGate  # noqa: F401


@dataclass
class SpinAlgebra:
    spin: float
    dim: int
    x: np.ndarray
    z: np.ndarray
    parity: np.ndarray


def spin_operators(spin: float) -> SpinAlgebra:
    """models.cpp:121-145 (ascending-m basis)."""
    two_s = 2.0 * spin
    if not (two_s >= 1.0) or abs(two_s - round(two_s)) > 1e-12:
        raise InvalidArgument("spin_operators: 2S must be a positive integer")
    d = int(round(two_s)) + 1
    x = np.zeros((d, d))
    z = np.zeros((d, d))
    par = np.zeros((d, d))
    for k in range(d):
        m = -spin + k
        z[k, k] = m
        par[k, k] = 1.0 if k % 2 == 0 else -1.0
        if k + 1 < d:
            v = 0.5 * np.sqrt(spin * (spin + 1.0) - m * (m + 1.0))
            x[k + 1, k] = v
            x[k, k + 1] = v
    return SpinAlgebra(spin, d, x, z, par)


@dataclass
class ChainModel:
    length: int = 2
    spin: float = 0.5
    field: float = 1.0


@dataclass
class CylinderModel:
    length: int = 4
    width: int = 2
    field: float = 3.0


Model = Union[ChainModel, CylinderModel]



def _pauli_x():
    return np.array([[0.0, 1.0], [1.0, 0.0]])


def _pauli_z():
    return np.array([[-1.0, 0.0], [0.0, 1.0]])


def _ring_component(op, i, w):
    out = np.eye(1)
    for k in range(w):
        out = np.kron(out, op if k == i else np.eye(2))
    return out


def _site_operators(model: Model):
    """models.cpp:62-98: (dim, charges, couplings [(a, b)], one_site)."""
    if isinstance(model, ChainModel):
        alg = spin_operators(model.spin)
        charges = [k % 2 for k in range(alg.dim)]
        s2 = model.spin * model.spin
        return alg.dim, charges, [(-(1.0 / s2) * alg.x, alg.x)], (model.field / model.spin) * alg.z
    if model.width < 2:
        raise InvalidArgument("cylinder: width must be >= 2")
    d = 1 << model.width
    charges = [bin(b).count("1") % 2 for b in range(d)]
    couplings = []
    for i in range(model.width):
        xi = _ring_component(_pauli_x(), i, model.width)
        couplings.append((-xi, xi))
    h = np.zeros((d, d))
    for i in range(model.width):
        h -= _ring_component(_pauli_x(), i, model.width) @ _ring_component(
            _pauli_x(), (i + 1) % model.width, model.width)
        h += model.field * _ring_component(_pauli_z(), i, model.width)
    return d, charges, couplings, h


def parity_structure(model: Model) -> SiteStructure:
    d, charges, _, _ = _site_operators(model)
    return SiteStructure(d, list(charges), sum(1 for q in charges if q == 0),
                         sum(1 for q in charges if q == 1))


def bond_hamiltonians(model: Model) -> List[np.ndarray]:
    """models.cpp:160-178: one-site terms split half/half (full at the ends)."""
    length = model.length
    if length < 2:
        raise InvalidArgument("bond_hamiltonians: need at least two sites")
    d, _, couplings, one = _site_operators(model)
    idm = np.eye(d)
    coupling = sum(np.kron(a, b) for a, b in couplings)
    out = []
    for b in range(length - 1):
        wl = 1.0 if b == 0 else 0.5
        wr = 1.0 if b + 2 == length else 0.5
        out.append(coupling + wl * np.kron(one, idm) + wr * np.kron(idm, one))
    return out





def _commutes_with_parity(h, charges):
    d = len(charges)
    for r in range(d * d):
        for c in range(d * d):
            if h[r, c] == 0.0:
                continue
            if (charges[r // d] ^ charges[r % d]) != (charges[c // d] ^ charges[c % d]):
                return False
    return True


def build_gate(h_bond: np.ndarray, site_charges: List[int], dt: float,
               form: GateForm = GateForm.block, schmidt_tol: float = 1e-14) -> TwoSiteGate:
    """models.cpp:180-247."""
    d = len(site_charges)
    h_bond = np.asarray(h_bond, dtype=np.float64)
    if h_bond.shape != (d * d, d * d):
        raise InvalidArgument("build_gate: h_bond must be d^2 x d^2")
    if not np.allclose(h_bond, h_bond.T, rtol=1e-12, atol=0.0):
        raise InvalidArgument("build_gate: h_bond must be symmetric")
    if not _commutes_with_parity(h_bond, site_charges):
        raise InvalidArgument("build_gate: h_bond must conserve parity")
    if not (dt >= 0.0):
        raise InvalidArgument("build_gate: dt must be >= 0")
    if not (0.0 < schmidt_tol < 1.0):
        raise InvalidArgument("build_gate: schmidt_tol must be in (0, 1)")
    w, v = np.linalg.eigh(h_bond)
    gate = TwoSiteGate(form, dt, (v * np.exp(-dt * w)[None, :]) @ v.T, [])
    if form != GateForm.product:
        return gate
    for q in (0, 1):
        pairs = [(mp, m) for mp in range(d) for m in range(d)
                 if (site_charges[mp] ^ site_charges[m]) == q]
        if not pairs:
            continue
        r = np.empty((len(pairs), len(pairs)))
        for i, (a0, a1) in enumerate(pairs):
            for j, (b0, b1) in enumerate(pairs):
                r[i, j] = gate.block[a0 * d + b0, a1 * d + b1]
        u, s, vt = np.linalg.svd(r)
        for k in range(len(s)):
            if s[k] <= 0.0:
                break
            left = np.zeros((d, d))
            right = np.zeros((d, d))
            root = np.sqrt(s[k])
            for i, (a0, a1) in enumerate(pairs):
                left[a0, a1] = root * u[i, k]
                right[a0, a1] = root * vt[k, i]
            gate.terms.append(KronTerm(left, right, q, float(s[k])))
    gate.terms.sort(key=lambda t: (-t.weight, t.charge))
    cut = schmidt_tol * gate.terms[0].weight if gate.terms else 0.0
    while gate.terms and gate.terms[-1].weight <= cut:
        gate.terms.pop()
    return gate
