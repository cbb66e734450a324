"""Interface types of the TEBD two-site bond update (rlftn models.hpp /
mps.hpp): the site structure (physical dimension, Z2 charges) and a two-site
gate in block or Kronecker-product form, as `apply_gate` (mps.cpp:111-323)
consumes them.  Building gates for a model (spin operators, Hamiltonians,
exp(-dt h)) is out of scope; the tests and tools construct them with
tests/tebd_models.py."""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np


@dataclass
class SiteStructure:
    """models.hpp SiteStructure: local dimension and the parity of each state."""
    dim: int
    charges: List[int]
    dim_even: int = 0
    dim_odd: int = 0


class GateForm(enum.Enum):
    """models.hpp GateForm: dense d^2 x d^2 block or a sum of Kronecker terms."""
    block = 0
    product = 1


@dataclass
class KronTerm:
    """One operator-Schmidt term left (x) right of a product-form gate."""
    left: np.ndarray
    right: np.ndarray
    charge: int = 0
    weight: float = 0.0


@dataclass
class TwoSiteGate:
    """models.hpp TwoSiteGate."""
    form: GateForm = GateForm.block
    dt: float = 0.0
    block: np.ndarray = None
    terms: List[KronTerm] = field(default_factory=list)
