"""paper_1402_3661_b200 -- B200-native Krylov SpMV over Z/lZ.

A from-scratch sm_100a build of the block-Wiedemann hot path of
arXiv:1402.3661 (reference package `sldlag`): the repeated exact sparse
matrix-vector product v <- A v mod l (160-650-bit primes) and the projected
sequence a_i = X^T A^i y.  Python keeps the reference's entry points and
plugin protocols; the arithmetic runs in hand-written CUDA kernels behind a
plain C ABI (include/sldb200.h, libsldb200.so).  No CPU fallback.
"""
from .modring import (
    TAG_FULL, TAG_MINUS_ONE, TAG_PLUS_ONE, TAG_SMALL, PrimeModulus, digit_count,
    ints_to_limbs, ints_to_planes, limbs_to_ints, limbs_to_planes, planes_to_ints,
    planes_to_limbs,
)
from .spmatrix import (
    DeviceKernel, SparseMatrix, classify, load_matrix, load_vector, spmv_planes, spmv_sequential,
    store_matrix, store_vector,
)
from .fileio import BadMagic, FormatError, TruncatedFile
from .checkpoint import CHECKPOINT_EVERY, CheckpointManager, HaltRequested, load_terms, store_terms
from .solver import (
    B200ChainGroup, B200Multiplier, BlockingParams, BlockSequence, DenseRows, SequentialMultiplier, UnitRows,
    draw_blocks, krylov_block, krylov_column, krylov_length, krylov_scalar,
    GeneratorFailure, KernelVector, SolverFailure, mksol_block, mksol_scalar, verify_kernel,
)

__version__ = "0.1.0"
