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
        return int(sum(np.count_nonzero(d) for d in self.dense))


class LazyFactors:
    """``factors`` of a device-built BlockCholesky: the sparse copy of each
    dense part factor (sp.csr_matrix(lb), factor.py:148) made on first access,
    so a build with 10^5 parts does not pay for scipy object construction
    unless the index is saved or inspected."""

    def __init__(self, dense):
        self._dense = dense
        self._cache = {}

    def __len__(self):
        return len(self._dense)

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        f = self._cache.get(b)
        if f is None:
            import scipy.sparse as sp

            f = self._cache[b] = sp.csr_matrix(self._dense[b])
        return f

    def __iter__(self):
        return (self[i] for i in range(len(self)))


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
