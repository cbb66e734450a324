"""B200-native randomized truncated SVD (RSVD) engine.

Drop-in for the factorization path of rlftn (arXiv 1710.01463's
TEBD bond compression): ``rsvd``, ``randomized_range``,
``reconstruction_error``, ``tsvd``, ``block_factorize``, the TEBD bond update
(``tebd.apply_gate`` / ``apply_gate_layer``) and the seed/RNG contract, computed by hand-written
sm_100a CUDA kernels in ``librsvd_b200.so`` behind the C ABI of
``include/rsvd_c.h``.
"""
from ._lib import DeviceError, Handle, InvalidArgument, LibraryMissing, NumericalError
from .factorize import (
    BatchedFactorization,
    ErrorNorm,
    RsvdParams,
    TruncatedFactorization,
    randomized_range,
    reconstruction_error,
    rsvd,
    rsvd_batched,
    tsvd,
    tsvd_batched,
)
from .blocks import (BlockDiagMatrix, BlockFactorization, BlockMethod, RankPolicy,
                     SectorRankRequest, block_factorize, block_factorize_many, sector_request)
from . import gates, matrix_io, tebd  # noqa: E402  (CLI: python -m paper_1710_01463_b200.cli)
from .rng import CounterRng, derive_seed, mix64, seed_tag

__all__ = [
    "BatchedFactorization", "CounterRng", "DeviceError", "ErrorNorm", "Handle", "InvalidArgument",
    "LibraryMissing", "NumericalError", "RsvdParams", "TruncatedFactorization", "derive_seed",
    "mix64", "randomized_range", "reconstruction_error", "rsvd", "rsvd_batched", "seed_tag",
    "tsvd", "tsvd_batched", "BlockDiagMatrix", "BlockFactorization", "BlockMethod", "RankPolicy",
    "SectorRankRequest", "block_factorize", "block_factorize_many", "sector_request", "gates",
    "tebd", "matrix_io",
]
