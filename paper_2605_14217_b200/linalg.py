"""Seeded constructors for adapter parameters (host side, registration only).

These build the float64 parameter bundles that are uploaded into the HBM
pool; they never run on the hot path.  They follow
pkg/src/prefillsim/linalg.py:27-69 step for step (same PCG64 streams, same
operation order), so `init_zero_delta(kind, r, dims, seed)` here produces
bit-identical arrays to the reference's — the parity tests rely on that.
"""

from __future__ import annotations

import numpy as np

from .errors import DomainError, RankError, ShapeError

__all__ = ["rng_from_seed", "kaiming_uniform", "random_orthonormal_rows"]


def rng_from_seed(seed: int, stream: int = 0) -> np.random.Generator:
    """PCG64 generator for (seed, stream)   (linalg.py:27-35)."""
    if seed < 0:
        raise DomainError(f"seed must be non-negative, got {seed}")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, stream))))


def kaiming_uniform(rows: int, cols: int, seed: int) -> np.ndarray:
    """U[-b, b], b = sqrt(6 / cols), fan-in = cols   (linalg.py:38-46)."""
    if rows < 1 or cols < 1:
        raise ShapeError(f"matrix dims must be positive, got {rows}x{cols}")
    bound = np.sqrt(6.0 / cols)
    return rng_from_seed(seed).uniform(-bound, bound, size=(rows, cols))


def random_orthonormal_rows(r: int, d: int, seed: int) -> np.ndarray:
    """(r, d) orthonormal rows: Gaussian draw + two MGS passes   (linalg.py:49-69)."""
    if r < 1:
        raise RankError(f"need at least one row, got r={r}")
    if r > d:
        raise RankError(f"cannot fit {r} orthonormal rows in dimension {d}")
    q = rng_from_seed(seed).normal(size=(r, d))
    for _ in range(2):
        for i in range(r):
            for j in range(i):
                q[i] -= (q[i] @ q[j]) * q[j]
            norm = np.linalg.norm(q[i])
            if norm == 0.0:
                raise RankError("degenerate draw while orthogonalising")
            q[i] /= norm
    return q
