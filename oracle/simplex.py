"""Polynomial fields on a simplex in barycentric form, in extended precision.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything the reference construction of P:581-807 needs reduces to integrals
of barycentric monomials over a simplex S of dimension l,
    int_S lambda^gamma = l! |S| gamma! / (|gamma| + l)!          (textbook)
and to the constant gradients g_k = grad lambda_k. A field is stored as
coefficients in a (redundant) barycentric frame:
  0-form  sum_gamma c_gamma lambda^gamma
  1-form  sum_{gamma,m} c_{gamma,m} lambda^gamma g_m
  2-form  sum_{gamma,(a<b)} c_{gamma,ab} lambda^gamma (g_a x g_b)
with Gram metrics G_km = g_k.g_m and H_(ab)(cd) = G_ac G_bd - G_ad G_bc.
Tangential traces onto a subsimplex s keep the terms with supp(gamma) and m
(or a,b) inside s (grad lambda_m is normal to s when m is not a vertex of s).
"""
from __future__ import annotations

import itertools
import math
from functools import lru_cache

import numpy as np

from .xprec import LD, ld, inv_ld, mm_ld


@lru_cache(maxsize=None)
def multi_indices(nv: int, q: int):
    """All gamma in N^nv with |gamma| = q, lexicographically descending, as an
    int64 array [N, nv]."""
    if nv == 1:
        return np.array([[q]], dtype=np.int64)
    rows = []
    for a in range(q, -1, -1):
        for rest in multi_indices(nv - 1, q - a):
            rows.append((a,) + tuple(rest))
    return np.array(rows, dtype=np.int64).reshape(-1, nv)


@lru_cache(maxsize=None)
def mi_lookup(nv: int, q: int):
    return {tuple(r): i for i, r in enumerate(multi_indices(nv, q))}


@lru_cache(maxsize=None)
def _fact_table(n: int = 64):
    return np.array([ld(math.factorial(k)) for k in range(n)], dtype=LD)


def pairs(nv: int):
    return [(a, b) for a in range(nv) for b in range(a + 1, nv)]


class Simplex:
    """An l-simplex given by Cartesian vertex coordinates (longdouble)."""

    def __init__(self, coords):
        c = np.array(coords, dtype=LD)
        self.coords = c
        self.nv = c.shape[0]
        self.l = self.nv - 1
        self.dim = c.shape[1]
        assert self.dim == self.l, "canonical simplices live in R^l"
        E = (c[1:] - c[0]).T  # dim x l, columns = edge vectors
        Einv = inv_ld(E)  # rows j-1 = grad lambda_j
        g = np.zeros((self.nv, self.dim), dtype=LD)
        g[1:] = Einv
        g[0] = -Einv.sum(axis=0)
        self.g = g
        det = _det_ld(E)
        self.vol = abs(det) / ld(math.factorial(self.l))
        self.G = g @ g.T
        pr = pairs(self.nv)
        self.pairs = pr
        H = np.zeros((len(pr), len(pr)), dtype=LD)
        for i, (a, b) in enumerate(pr):
            for j, (cc, d) in enumerate(pr):
                H[i, j] = self.G[a, cc] * self.G[b, d] - self.G[a, d] * self.G[b, cc]
        self.H = H

    # ---------------------------------------------------------------- integrals
    def I(self, q1: int, q2: int) -> np.ndarray:
        """I[a,b] = int_S lambda^(gamma_a + gamma_b), gamma_a in MI(q1), gamma_b in MI(q2)."""
        A = multi_indices(self.nv, q1)
        B = multi_indices(self.nv, q2)
        f = _fact_table()
        S = A[:, None, :] + B[None, :, :]
        num = np.prod(f[S], axis=2)
        return num * (ld(math.factorial(self.l)) * self.vol / f[q1 + q2 + self.l])

    def mass0(self, F1, q1, F2, q2):
        return mm_ld(mm_ld(F1, self.I(q1, q2)), F2.T)

    def mass1(self, F1, q1, F2, q2):
        T = np.kron(self.I(q1, q2), self.G)
        return mm_ld(mm_ld(F1, T), F2.T)

    def mass2(self, F1, q1, F2, q2):
        T = np.kron(self.I(q1, q2), self.H)
        return mm_ld(mm_ld(F1, T), F2.T)

    # ---------------------------------------------------------------- operators
    def grad_op(self, q: int) -> np.ndarray:
        """Matrix mapping 0-form coefficients (deg q, as a row) to 1-form (deg q-1)."""
        nv = self.nv
        A = multi_indices(nv, q)
        lk = mi_lookup(nv, q - 1) if q > 0 else {}
        Dm = np.zeros((len(A), max(len(lk), 1) * nv if q > 0 else 0), dtype=LD)
        for i, a in enumerate(A):
            for m in range(nv):
                if a[m] > 0:
                    b = list(a)
                    b[m] -= 1
                    Dm[i, lk[tuple(b)] * nv + m] += a[m]
        return Dm

    def curl_op(self, q: int) -> np.ndarray:
        """1-form (deg q) -> 2-form (deg q-1): curl(lambda^gamma g_m) = sum_k gamma_k lambda^(gamma-e_k) g_k x g_m."""
        nv = self.nv
        A = multi_indices(nv, q)
        lk = mi_lookup(nv, q - 1)
        pr = {p: i for i, p in enumerate(self.pairs)}
        npair = len(self.pairs)
        C = np.zeros((len(A) * nv, len(lk) * npair), dtype=LD)
        for i, a in enumerate(A):
            for m in range(nv):
                for k in range(nv):
                    if a[k] == 0 or k == m:
                        continue
                    b = list(a)
                    b[k] -= 1
                    if k < m:
                        C[i * nv + m, lk[tuple(b)] * npair + pr[(k, m)]] += a[k]
                    else:
                        C[i * nv + m, lk[tuple(b)] * npair + pr[(m, k)]] -= a[k]
        return C

    def whitney_products(self, elems, q: int) -> np.ndarray:
        """Rows = 1-form coefficients (deg q+1) of lambda^alpha w_ij,
        w_ij = lambda_i g_j - lambda_j g_i, for (alpha, i, j) in elems, |alpha| = q."""
        nv = self.nv
        lk = mi_lookup(nv, q + 1)
        F = np.zeros((len(elems), len(lk) * nv), dtype=LD)
        for r, (alpha, i, j) in enumerate(elems):
            ai = list(alpha)
            ai[i] += 1
            aj = list(alpha)
            aj[j] += 1
            F[r, lk[tuple(ai)] * nv + j] += 1
            F[r, lk[tuple(aj)] * nv + i] -= 1
        return F

    def whitney2_products(self, elems, q: int) -> np.ndarray:
        """Rows = 2-form coefficients (deg q+1, pair frame) of lambda^alpha w_ijk,
        w_ijk = lambda_i g_j x g_k - lambda_j g_i x g_k + lambda_k g_i x g_j
        (the Whitney 2-form of face ijk up to the factor 2), (alpha, i, j, k) in
        elems with i < j < k, |alpha| = q."""
        lk = mi_lookup(self.nv, q + 1)
        pr = {p: i for i, p in enumerate(self.pairs)}
        npair = len(self.pairs)
        F = np.zeros((len(elems), len(lk) * npair), dtype=LD)
        for r, (alpha, i, j, k) in enumerate(elems):
            for m, pair, sgn in ((i, (j, k), 1), (j, (i, k), -1), (k, (i, j), 1)):
                a = list(alpha)
                a[m] += 1
                F[r, lk[tuple(a)] * npair + pr[pair]] += sgn
        return F

    def div_op(self, q: int) -> np.ndarray:
        """2-form (deg q, pair frame, 3D proxy g_a x g_b) -> 0-form (deg q-1):
        div(lambda^gamma g_a x g_b) = sum_k gamma_k lambda^(gamma-e_k) g_k . (g_a x g_b)."""
        assert self.dim == 3
        nv = self.nv
        A = multi_indices(nv, q)
        lk = mi_lookup(nv, q - 1)
        npair = len(self.pairs)
        D = np.zeros((len(A) * npair, len(lk)), dtype=LD)
        for i, a in enumerate(A):
            for pi, (pa, pb) in enumerate(self.pairs):
                cr = np.cross(self.g[pa], self.g[pb])
                for k in range(nv):
                    if a[k] == 0 or k in (pa, pb):
                        continue
                    b = list(a)
                    b[k] -= 1
                    D[i * npair + pi, lk[tuple(b)]] += a[k] * (self.g[k] @ cr)
        return D

    # ---------------------------------------------------------------- evaluation
    def bary(self, x) -> np.ndarray:
        """Barycentric coordinates of Cartesian points x [npts, dim]."""
        x = np.asarray(x, dtype=LD)
        lam = (x - self.coords[0]) @ self.g[1:].T
        out = np.empty((x.shape[0], self.nv), dtype=LD)
        out[:, 1:] = lam
        out[:, 0] = 1 - lam.sum(axis=1)
        return out

    def cart(self, bary) -> np.ndarray:
        return np.asarray(bary, dtype=LD) @ self.coords

    def monomials(self, bary, q: int) -> np.ndarray:
        """[npts, N_q] values of lambda^gamma."""
        A = multi_indices(self.nv, q)
        bary = np.asarray(bary, dtype=LD)
        return np.prod(bary[:, None, :] ** A[None, :, :], axis=2)

    def eval0(self, F, q, bary):
        """F [nf, N_q] -> values [npts, nf]."""
        return mm_ld(self.monomials(bary, q), F.T)

    def eval1(self, F, q, bary):
        """F [nf, N_q*nv] -> Cartesian vectors [npts, nf, dim]:
        sum_a lambda^a(x) sum_m F[f, a, m] g_m (the 1-form's proxy)."""
        Mo = self.monomials(bary, q)
        Fr = F.reshape(F.shape[0], -1, self.nv)
        return self._contract(Mo, Fr @ self.g.astype(LD))

    def eval2(self, F, q, bary):
        """F [nf, N_q*npairs] -> curl values: [npts, nf, 3] in 3D, [npts, nf] in 2D."""
        Mo = self.monomials(bary, q)
        Fr = F.reshape(F.shape[0], -1, len(self.pairs))
        if self.dim == 3:
            cr = np.array([np.cross(self.g[a].astype(LD), self.g[b].astype(LD)) for a, b in self.pairs], dtype=LD)
            return self._contract(Mo, Fr @ cr)
        if self.dim == 2:
            cr = np.array([self.g[a][0] * self.g[b][1] - self.g[a][1] * self.g[b][0] for a, b in self.pairs], dtype=LD)
            return self._contract(Mo, (Fr @ cr)[:, :, None])[:, :, 0]
        raise ValueError("no curl in 1D")

    @staticmethod
    def _contract(Mo, H):
        """out[p, f, d] = sum_a Mo[p, a] H[f, a, d] (values of the monomial
        expansion; the sum over the form's frame is already in H)."""
        nf, na, nd = H.shape
        Ht = np.ascontiguousarray(np.transpose(H, (1, 0, 2)).reshape(na, nf * nd))
        return mm_ld(Mo, Ht).reshape(Mo.shape[0], nf, nd)


def _det_ld(E):
    n = E.shape[0]
    if n == 1:
        return E[0, 0]
    if n == 2:
        return E[0, 0] * E[1, 1] - E[0, 1] * E[1, 0]
    if n == 3:
        return (E[0, 0] * (E[1, 1] * E[2, 2] - E[1, 2] * E[2, 1])
                - E[0, 1] * (E[1, 0] * E[2, 2] - E[1, 2] * E[2, 0])
                + E[0, 2] * (E[1, 0] * E[2, 1] - E[1, 1] * E[2, 0]))
    raise ValueError


# --------------------------------------------------------------------------
# Reference geometry (DESIGN.md R-A1/R-A2): edge length 2, centroid at origin.
def _s(x):
    return np.sqrt(LD(x))


def reference_tet() -> Simplex:
    """T-hat: V0=(-1,-1/sqrt3,-1/sqrt6), V1=(1,-1/sqrt3,-1/sqrt6),
    V2=(0,2/sqrt3,-1/sqrt6), V3=(0,0,3/sqrt6)."""
    s3, s6 = _s(3), _s(6)
    return Simplex([[-1, -1 / s3, -1 / s6], [1, -1 / s3, -1 / s6], [0, 2 / s3, -1 / s6], [0, 0, 3 / s6]])


def canonical_face() -> Simplex:
    s3 = _s(3)
    return Simplex([[-1, -1 / s3], [1, -1 / s3], [0, 2 / s3]])


def canonical_edge() -> Simplex:
    return Simplex([[-1], [1]])


def canonical(l: int) -> Simplex:
    return {1: canonical_edge, 2: canonical_face, 3: reference_tet}[l]()


# Local subsimplices of T-hat (sorted local vertex lists), DESIGN.md R-A8 order.
TET_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
TET_FACES = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)]


def restrict_mi(q: int, nv_parent: int, s) -> tuple[np.ndarray, np.ndarray]:
    """For parent multi-indices of degree q: (mask of those supported on s,
    their index in the child's MI(q) list)."""
    A = multi_indices(nv_parent, q)
    s = list(s)
    others = [k for k in range(nv_parent) if k not in s]
    ok = np.all(A[:, others] == 0, axis=1) if others else np.ones(len(A), dtype=bool)
    lk = mi_lookup(len(s), q)
    idx = np.array([lk[tuple(a[s])] if o else -1 for a, o in zip(A, ok)], dtype=np.int64)
    return ok, idx


def trace0(F, q, nv_parent, s):
    """Trace of 0-forms (rows of F, deg q) onto subsimplex s (child numbering = position in s)."""
    ok, idx = restrict_mi(q, nv_parent, s)
    out = np.zeros((F.shape[0], len(multi_indices(len(s), q))), dtype=LD)
    for a in np.nonzero(ok)[0]:
        out[:, idx[a]] += F[:, a]
    return out


def trace2(F, q, nv_parent, s):
    """Trace of 2-forms (rows of F, deg q, pair frame) onto subsimplex s: the
    terms with supp(gamma) and both pair vertices inside s (d lambda_m vanishes
    tangentially for m not in s), in the child's pair frame."""
    ok, idx = restrict_mi(q, nv_parent, s)
    s = list(s)
    pp, cp = pairs(nv_parent), {p: i for i, p in enumerate(pairs(len(s)))}
    npp, npc = len(pp), len(cp)
    out = np.zeros((F.shape[0], len(multi_indices(len(s), q)) * npc), dtype=LD)
    for a in np.nonzero(ok)[0]:
        for pi, (x, y) in enumerate(pp):
            if x in s and y in s:
                out[:, idx[a] * npc + cp[(s.index(x), s.index(y))]] += F[:, a * npp + pi]
    return out


def trace1(F, q, nv_parent, s):
    """Tangential trace of 1-forms (rows of F, deg q) onto subsimplex s."""
    ok, idx = restrict_mi(q, nv_parent, s)
    s = list(s)
    nvc = len(s)
    out = np.zeros((F.shape[0], len(multi_indices(nvc, q)) * nvc), dtype=LD)
    for a in np.nonzero(ok)[0]:
        for cm, m in enumerate(s):
            out[:, idx[a] * nvc + cm] += F[:, a * nv_parent + m]
    return out
