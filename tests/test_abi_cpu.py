"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/rsvd_c.h declares, validates arguments with the reference's
messages (factorize.cpp:79-83, 56-59) and fails cleanly without a device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsvd_c.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rsvd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_core_entry_points():
    syms = declared_symbols()
    for s in ("rsvd_create", "rsvd_destroy", "rsvd_f64", "rsvd_f64_batched",
              "rsvd_randomized_range_f64", "rsvd_fill_gaussian_f64", "rsvd_last_error",
              "rsvd_reconstruction_error_f64", "rsvd_validate_params"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1710_01463_b200 import _lib

    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding table covers the header exactly
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_host_only_entry_points():
    from paper_1710_01463_b200 import _lib, rng

    lib = _lib.load()
    assert lib.rsvd_version().startswith(b"rsvd_b200")
    for z in (0, 1, 2, 3, 2**63 + 5):
        assert lib.rsvd_mix64(z) == rng.mix64(z)
        assert lib.rsvd_derive_seed(z, 7) == rng.derive_seed(z, 7)


@pytest.mark.parametrize(
    "args,msg",
    [
        ((0, 5, 1, 0, 4), "rsvd: empty matrix"),
        ((5, 0, 1, 0, 4), "rsvd: empty matrix"),
        ((4, 4, 0, 0, 4), "rsvd: rank must be >= 1"),
        ((4, 4, 3, 2, 4), "rsvd: oversample must be >= rank"),
        ((4, 4, 3, 5, 4), "randomized_range: need 1 <= ell <= min(m, n)"),
        ((4, 4, 10, 0, 4), "rsvd: oversample must be >= rank"),  # ell = min(20, 4) < 10
        ((4, 4, 2, 0, -1), "randomized_range: power must be >= 0"),
    ],
)
def test_validation_messages(args, msg):
    from paper_1710_01463_b200 import _lib

    with pytest.raises(_lib.InvalidArgument) as e:
        _lib.validate_params(*args)
    assert str(e.value) == msg


def test_validation_resolves_default_ell():
    from paper_1710_01463_b200 import _lib

    assert _lib.validate_params(100, 80, 10, 0, 4) == 20
    assert _lib.validate_params(100, 15, 10, 0, 4) == 15  # clipped to min(m, n)
    assert _lib.validate_params(100, 80, 10, 12, 0) == 12


def test_no_device_fails_loudly_without_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1710_01463_b200 import DeviceError, RsvdParams, rsvd

    with pytest.raises(DeviceError):
        rsvd(np.eye(8), RsvdParams(2, 4, 1, 3))


def test_missing_library_raises(monkeypatch, tmp_path):
    from paper_1710_01463_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.LibraryMissing):
        _lib.load()
