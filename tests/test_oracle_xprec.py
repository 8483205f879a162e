"""Pins for the oracle's extended-precision primitives (oracle/xprec.py)."""
import numpy as np
import mpmath

from oracle.xprec import LD, eigh_ld, solve_ld, qr_pos_ld, ld
from fractions import Fraction


def _sym_with_clusters(n, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.sort(rng.uniform(0.1, 10, n))
    w[3:6] = w[3]           # exact triple cluster
    w[8] = w[7] * (1 + 1e-6)  # near-degenerate pair
    return (Q * w) @ Q.T, w


def test_eigh_ld_residual_and_orthogonality():
    A, w_true = _sym_with_clusters(30, 0)
    A = A.astype(LD)
    w, X = eigh_ld(A)
    R = A @ X - X * w[None, :]
    assert float(np.abs(R).max()) < 1e-16 * float(np.abs(A).max())
    O = X.T @ X - np.eye(30, dtype=LD)
    assert float(np.abs(O).max()) < 1e-17


def test_eigh_ld_against_mpmath():
    rng = np.random.default_rng(1)
    B = rng.standard_normal((8, 8))
    A = B + B.T
    mpmath.mp.dps = 40
    E, _ = mpmath.eigsy(mpmath.matrix(A.tolist()))
    ref = sorted(float(E[i]) for i in range(8))
    w, _ = eigh_ld(A.astype(LD))
    # compare in longdouble against the 40-digit values
    Es = sorted([E[i] for i in range(8)])
    for a, b in zip(w, Es):
        assert abs(float(a - LD(str(b)))) < 1e-17 * max(1.0, abs(float(b)))


def test_eigh_ld_rank_deficient_gram():
    rng = np.random.default_rng(2)
    B = rng.standard_normal((20, 12))
    M = (B @ B.T).astype(LD)          # rank 12
    w, X = eigh_ld(M)
    assert int((w > 1e-13 * w.max()).sum()) == 12


def test_solve_ld_against_mpmath():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((7, 7))
    b = rng.standard_normal(7)
    mpmath.mp.dps = 40
    xr = mpmath.lu_solve(mpmath.matrix(A.tolist()), mpmath.matrix(b.tolist()))
    x = solve_ld(A.astype(LD), b.astype(LD))
    for i in range(7):
        assert abs(float(x[i] - LD(str(xr[i])))) < 1e-16 * max(1.0, abs(float(xr[i])))


def test_qr_pos():
    rng = np.random.default_rng(4)
    P = rng.standard_normal((4, 4)).astype(LD)
    Q, R = qr_pos_ld(P)
    assert np.all(np.diag(R) > 0)
    assert float(np.abs(Q @ R - P).max()) < 1e-17
    assert float(np.abs(np.tril(R, -1)).max()) == 0.0


def test_ld_conversion_exact():
    assert ld(Fraction(1, 3)) == LD(1) / LD(3)
    big = 27 * 10 ** 25
    assert abs(float(ld(big) / LD("2.7e26") - 1)) < 1e-18


def test_mm_ld_bitwise_equal_to_numpy_and_exact_on_integers():
    """oracle/ldgemm.c (mm_ld) is numpy's non-BLAS longdouble matmul loop spread
    over threads: bitwise equal on random operands (contiguous and transposed
    views, ragged shapes), and exact on small-integer products (every partial
    sum representable) against Python integers."""
    from oracle.xprec import mm_ld
    rng = np.random.default_rng(7)
    for m, k, n in [(37, 53, 41), (64, 64, 64), (5, 300, 3), (130, 7, 90)]:
        A = rng.standard_normal((m, k)).astype(LD) / LD(3)
        B = rng.standard_normal((k, n)).astype(LD) / LD(7)
        assert np.array_equal(mm_ld(A, B), A @ B)
        At = np.ascontiguousarray(A.T)
        assert np.array_equal(mm_ld(At.T, B), A @ B)
    Ai = rng.integers(-1000, 1000, (40, 60))
    Bi = rng.integers(-1000, 1000, (60, 50))
    exact = np.array([[sum(int(Ai[i, l]) * int(Bi[l, j]) for l in range(60)) for j in range(50)] for i in range(40)])
    assert np.array_equal(mm_ld(Ai.astype(LD), Bi.astype(LD)).astype(np.int64), exact)
