"""Factor data types of the KLRC index (the query-time half of factor.py).

These mirror the reference's containers (factor.py:58-219) so a loaded index
looks like the reference's KatzIndex; the arithmetic they carry is done on
the GPU by lrc.cu, not by these classes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class FactorizationError(RuntimeError):
    """A pivot failed; the block is not positive definite (factor.py:23-24)."""


class SpectrumError(RuntimeError):
    """Correction eigenvalues left [0, 1) (factor.py:27-28)."""


@dataclass(eq=False)
class BlockCholesky:
    """Per-part factors of the block-diagonal interior block (factor.py:58-86).

    block_offsets delimit parts; orders[b] is the local fill-reducing order
    of part b and factors[b] its sparse lower-triangular factor.
    """

    block_offsets: np.ndarray
    orders: list
    factors: list
    dense: list = field(default=None, repr=False)

    def __post_init__(self):
        if self.dense is None:
            self.dense = [f.toarray() for f in self.factors]

    @property
    def n(self):
        return int(self.block_offsets[-1])

    @property
    def num_blocks(self):
        return len(self.factors)

    @property
    def nnz(self):
        return int(sum(f.nnz for f in self.factors))


@dataclass(eq=False)
class DenseCholesky:
    """Dense lower factor L of the separator block, M22 = L L' (factor.py:155-168)."""

    factor: np.ndarray

    def __post_init__(self):
        self.factor = np.asfortranarray(self.factor, dtype=np.float64)

    @property
    def n(self):
        return self.factor.shape[0]


@dataclass(eq=False)
class LowRankCorrection:
    """Top eigenpairs (U, sigma) of R = L^-1 M12' M11^-1 M12 L^-T (factor.py:205-219)."""

    ell: int
    vectors: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.vectors = np.asfortranarray(self.vectors, dtype=np.float64)
