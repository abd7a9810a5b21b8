"""Input contract and seeded input recipes for the condensation path.

Mirrors the storage contract of the reference (``as_matrix`` /
``require_square``, /root/reference/pkg/src/mcnd/matrix.py:32-48): inputs are
coerced to C-contiguous float64, must be 2-D, non-empty, finite and square,
and violations raise ``ValueError`` with the same messages.

The generator kinds restate the reference's seeded recipes
(matrix.py:69-106) so the parity tests feed the GPU and the oracle the exact
bytes the reference would have built; the BASELINE configs C1..C5 follow
SURVEY.md §8(d).  Only numpy PCG64 is used, so BLAS-free recipes are
bit-reproducible on any host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GENERATOR_KINDS = (
    "uniform-random",
    "diagonally-dominant",
    "scaled-correlation",
    "identity",
    "singular-planted",
)


def as_matrix(data) -> np.ndarray:
    """matrix.py:32-41: canonical C-contiguous float64 2-D finite matrix."""
    a = np.ascontiguousarray(data, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got {a.ndim}-D")
    if a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("matrix dimensions must be positive")
    if not np.isfinite(a).all():
        raise ValueError("matrix entries must be finite (no NaN/Inf)")
    return a


def require_square(a) -> np.ndarray:
    """matrix.py:44-48."""
    a = as_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise ValueError(f"matrix must be square, got {a.shape}")
    return a


def square_for_device(data) -> np.ndarray:
    """require_square without the O(N^2) host finiteness scan: the CUDA
    prologue checks finiteness while copying (k1_condense.cu) and the call
    raises the same ValueError.  Non-square input still reports non-finite
    entries first, in the reference's check order (matrix.py:35-47)."""
    a = np.ascontiguousarray(data, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got {a.ndim}-D")
    if a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("matrix dimensions must be positive")
    if a.shape[0] != a.shape[1]:
        if not np.isfinite(a).all():
            raise ValueError("matrix entries must be finite (no NaN/Inf)")
        raise ValueError(f"matrix must be square, got {a.shape}")
    return a


@dataclass(frozen=True)
class MatrixSpec:
    """matrix.py:51-66: deterministic recipe (size, kind, seed)."""

    size: int
    kind: str
    seed: int = 0

    def __post_init__(self):
        if self.size < 1:
            raise ValueError("invalid size: must be >= 1")
        if self.kind not in GENERATOR_KINDS:
            raise ValueError(
                f"unknown generator kind {self.kind!r}; expected one of {GENERATOR_KINDS}")


def generate(spec: MatrixSpec) -> np.ndarray:
    """Seeded test matrices, same draws as matrix.py:69-106."""
    n, rng = spec.size, np.random.default_rng(spec.seed)
    kind = spec.kind
    if kind == "identity":
        return np.eye(n)
    if kind == "uniform-random":
        return rng.uniform(-1.0, 1.0, size=(n, n))
    if kind == "diagonally-dominant":
        a = rng.uniform(-1.0, 1.0, size=(n, n))
        a[np.diag_indices(n)] += float(n)
        return a
    if kind == "scaled-correlation":
        x = rng.normal(size=(n, n))
        g = x @ x.T / n + 0.5 * np.eye(n)
        g = (g + g.T) / 2.0
        d = np.sqrt(np.diag(g))
        s = np.where(np.arange(n) % 2 == 0, np.sqrt(2.0), 1e-5)
        return (g / np.outer(d, d)) * np.outer(s, s)
    if kind == "singular-planted":
        if n == 1:
            return np.zeros((1, 1))
        a = rng.uniform(-1.0, 1.0, size=(n, n))
        a[n // 2] = a[0]
        return a
    raise AssertionError(kind)


# --------------------------------------------------------------------------
# BASELINE.json configs; synthetic, seeded.
# --------------------------------------------------------------------------

def config_dense_normal(n: int = 1000, seed: int = 1) -> np.ndarray:
    """C1: iid N(0,1) (BLAS-free, bit-reproducible)."""
    return np.random.default_rng(seed).standard_normal((n, n))


def config_uniform(n: int = 8000, seed: int = 3) -> np.ndarray:
    """C3: iid U[-1,1]; identical to generate(MatrixSpec(n,'uniform-random',seed))."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))


def config_spd(n: int = 4000, seed: int = 2, ridge: float = 1e-3, k_mult: int = 2) -> np.ndarray:
    """C2: A = X X^T / (k n) + ridge*I, X in R^{n x kn} iid N(0,1).

    The Gram product goes through BLAS, so the bytes are host-dependent: tests
    always hand the very same array to the GPU and to the oracle."""
    x = np.random.default_rng(seed).standard_normal((n, k_mult * n))
    a = x @ x.T / (k_mult * n)
    a[np.diag_indices(n)] += ridge
    return a


def config_batched_spd(batch: int = 4096, n: int = 64, seed: int = 4, ridge: float = 1e-2) -> np.ndarray:
    """C4: A_b = X_b X_b^T / (2n) + ridge*I, X_b in R^{n x 2n} iid N(0,1)."""
    x = np.random.default_rng(seed).standard_normal((batch, n, 2 * n))
    a = np.matmul(x, x.transpose(0, 2, 1)) / (2 * n)
    a[:, np.arange(n), np.arange(n)] += ridge
    return a


def config_spd_device(n: int = 32768, seed: int = 5, ridge: float = 1e-2, device: str = "cuda"):
    """C5: A = X X^T / N + ridge*I with X in R^{N x N} iid N(0,1), generated on the
    GPU by a seeded torch CUDA generator (row blocks of X are consumed in order,
    i.e. "blockwise from a seed"); the Gram product is one DGEMM.  Returns a
    float64 CUDA tensor (8.6 GB at N=32768)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn((n, n), dtype=torch.float64, device=device, generator=g)
    a = x @ x.T
    del x
    a /= n
    a.diagonal().add_(ridge)
    return a
