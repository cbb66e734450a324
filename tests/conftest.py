import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    oracle.set_threads(min(os.cpu_count() or 1, 16))
    return oracle


@pytest.fixture(scope="session")
def golden_small():
    import numpy as np

    return np.load(os.path.join(ROOT, "tests", "golden", "rsvd_small.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def ref_mod():
    """The reference's own factorize.cpp / lapack.cpp / blocks.cpp, compiled
    unmodified into oracle/_ref/librlftn_ref.so (oracle/Makefile `ref`).  The
    parity anchor: missing it is a failure, not a skip."""
    from oracle import ref

    if not ref.available():
        from oracle import oracle

        oracle.build()
    if not ref.available():
        pytest.fail("oracle/_ref/librlftn_ref.so is missing: run `make -C oracle ref` "
                    "where /root/reference exists (build() does)")
    ref.set_threads(min(os.cpu_count() or 1, 16))
    return ref
