"""Extended-precision (x87 80-bit, numpy.longdouble) dense linear algebra.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper computes its bubble eigenbases "numerically ... offline"
without stating a precision; reading R-A24 fixes that the reference
element is built in extended precision and rounded to FP64 once. numpy.linalg
does not support longdouble, so the three primitives needed are written here:
  * eigh_ld  - symmetric eigendecomposition: LAPACK float64 start, then
               Ogita-Aishima refinement (RefSyEv) iterated in longdouble;
  * solve_ld - Gaussian elimination with partial pivoting in longdouble;
  * qr_pos_ld - modified Gram-Schmidt QR with positive diag(R).
Pinned in tests/test_oracle_xprec.py against residuals and mpmath.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
from fractions import Fraction

LD = np.longdouble

_HERE = os.path.dirname(os.path.abspath(__file__))
_LDGEMM_SO = os.path.join(_HERE, "_ldgemm.so")
_ldgemm = None


def build_ldgemm() -> str:
    """Compile oracle/ldgemm.c (the long-double product, OpenMP over rows)."""
    src = os.path.join(_HERE, "ldgemm.c")
    tmp = _LDGEMM_SO + f".{os.getpid()}.tmp"
    subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src], check=True)
    os.replace(tmp, _LDGEMM_SO)
    return _LDGEMM_SO


def _lib():
    global _ldgemm
    if _ldgemm is None:
        src = os.path.join(_HERE, "ldgemm.c")
        try:
            if not os.path.exists(_LDGEMM_SO) or os.path.getmtime(_LDGEMM_SO) < os.path.getmtime(src):
                build_ldgemm()
            lib = ctypes.CDLL(_LDGEMM_SO)
            lib.ld_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3
            lib.ld_gemm.restype = None
            _ldgemm = lib
        except (OSError, subprocess.CalledProcessError):
            _ldgemm = False  # no compiler: numpy's own (identical, slower) loop
    return _ldgemm


def mm_ld(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """A @ B in longdouble, bitwise equal to numpy's non-BLAS matmul (k summed in
    ascending order from 0), computed by oracle/ldgemm.c with the rows spread
    over the host's cores (numpy's longdouble loop is single-threaded)."""
    A = np.asarray(A, dtype=LD)
    B = np.asarray(B, dtype=LD)
    if A.ndim != 2 or B.ndim != 2:
        return A @ B
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise ValueError(f"mm_ld: shapes {A.shape} {B.shape}")
    lib = _lib()
    if not lib or m * k * n < 32768:
        return A @ B
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    C = np.empty((m, n), dtype=LD)
    lib.ld_gemm(A.ctypes.data, B.ctypes.data, C.ctypes.data, m, k, n)
    return C


def ld(x) -> np.longdouble:
    """Exact-as-possible conversion of int / Fraction / str to longdouble."""
    if isinstance(x, Fraction):
        return ld(x.numerator) / ld(x.denominator)
    if isinstance(x, int):
        # split so that each part is exactly representable
        neg = x < 0
        x = -x if neg else x
        acc = LD(0)
        scale = LD(1)
        while x:
            acc += LD(x & 0xFFFFFFFF) * scale
            scale *= LD(4294967296)
            x >>= 32
        return -acc if neg else acc
    return LD(x)


def eigh_ld(A: np.ndarray, iters: int = 4):
    """Symmetric eigendecomposition A = X diag(w) X^T in longdouble.

    w ascending. Start from float64 LAPACK (numpy.linalg.eigh), then apply the
    Ogita-Aishima refinement (SIAM J. Sci. Comput. 2018, Alg. 1):
      R = I - X^T X, S = X^T A X, w_i = s_ii / (1 - r_ii),
      E_ij = (s_ij + w_j r_ij) / (w_j - w_i)  if |w_i - w_j| > delta,
             r_ij / 2                         otherwise,
      X <- X + X E.
    Eigenvalues closer than delta_ij = max(1e-12 max(|w_i|,|w_j|), 1e-15 max|w|)
    are treated as a cluster: the refinement keeps X orthonormal on it but leaves the rotation
    inside the cluster free; callers canonicalize clusters (DESIGN.md R-A6).
    """
    A = np.asarray(A, dtype=LD)
    A = (A + A.T) / 2
    n = A.shape[0]
    if n == 0:
        return np.zeros(0, dtype=LD), np.zeros((0, 0), dtype=LD)
    w64, X64 = np.linalg.eigh(A.astype(np.float64))
    X = X64.astype(LD)
    I = np.eye(n, dtype=LD)
    for _ in range(iters):
        R = I - mm_ld(X.T, X)
        R = (R + R.T) / 2
        S = mm_ld(mm_ld(X.T, A), X)
        S = (S + S.T) / 2
        w = np.diag(S) / (1 - np.diag(R))
        scale = np.max(np.abs(w)) if n else LD(1)
        aw = np.abs(w)
        delta = np.maximum(LD(1e-12) * np.maximum(aw[:, None], aw[None, :]), LD(1e-15) * scale)
        D = w[None, :] - w[:, None]  # D_ij = w_j - w_i
        big = np.abs(D) > delta
        E = np.where(big, (S + w[None, :] * R) / np.where(big, D, 1), R / 2)
        X = X + mm_ld(X, E)
    R = I - mm_ld(X.T, X)
    S = mm_ld(mm_ld(X.T, A), X)
    w = np.diag(S) / (1 - np.diag(R))
    order = np.argsort(w.astype(np.float64), kind="stable")
    return w[order], X[:, order]


def solve_ld(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Solve A X = B by Gaussian elimination with partial pivoting (longdouble)."""
    A = np.array(A, dtype=LD, copy=True)
    B = np.array(B, dtype=LD, copy=True)
    vec = B.ndim == 1
    if vec:
        B = B[:, None]
    n = A.shape[0]
    for k in range(n):
        piv = k + int(np.argmax(np.abs(A[k:, k].astype(np.float64))))
        if A[piv, k] == 0:
            raise np.linalg.LinAlgError("singular matrix in solve_ld")
        if piv != k:
            A[[k, piv]] = A[[piv, k]]
            B[[k, piv]] = B[[piv, k]]
        f = A[k + 1:, k] / A[k, k]
        A[k + 1:, k:] -= f[:, None] * A[k, k:][None, :]
        B[k + 1:] -= f[:, None] * B[k][None, :]
    X = np.zeros_like(B)
    for k in range(n - 1, -1, -1):
        X[k] = (B[k] - A[k, k + 1:] @ X[k + 1:]) / A[k, k]
    return X[:, 0] if vec else X


def inv_ld(A: np.ndarray) -> np.ndarray:
    return solve_ld(A, np.eye(A.shape[0], dtype=LD))


def qr_pos_ld(A: np.ndarray):
    """A = Q R with Q orthonormal columns and diag(R) > 0 (modified Gram-Schmidt,
    two passes for stability). A is m x c with full column rank."""
    A = np.array(A, dtype=LD)
    m, c = A.shape
    Q = np.zeros((m, c), dtype=LD)
    R = np.zeros((c, c), dtype=LD)
    for j in range(c):
        v = A[:, j].copy()
        for _ in range(2):
            for i in range(j):
                r = Q[:, i] @ v
                R[i, j] += r
                v = v - r * Q[:, i]
        R[j, j] = np.sqrt(v @ v)
        Q[:, j] = v / R[j, j]
    return Q, R
