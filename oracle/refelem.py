"""The paper's reference elements CG_p, Ned1_p and RT_p on the equilateral T-hat.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper in its order:
  1. bubble spaces on the canonical edge / face / cell (Eq. 3.1);
  2. the augmented eigenproblem Eq. 3.9 on the whole bubble space,
     zero modes dropped, survivors renormalised to Eq. 3.8:
     (d psi_i, d psi_j) = delta_ij, (psi_i, psi_j) = lambda_j delta_ij;
     ordering / cluster canonicalization by DESIGN.md R-A5..A7;
  3. the dofs of §3.4.1 (Eq. 3.14), §3.4.2 (Eq. 3.16) and
     §3.4.3 (Eq. 3.18; the Psi are Ned1_p's, DESIGN.md R-D1),
     with the canonical eigenbases carried to the subsimplices of T-hat by the
     vertex-order-preserving isometry (R-A2; in barycentric form this is a
     relabelling of vertices);
  4. the Ciarlet dual basis l_i(phi_j) = delta_ij by inverting the
     Vandermonde matrix in extended precision (R-A24).
Polynomial spans: CG_p = P_p in the scaled Bernstein basis (p!/beta!) lambda^beta;
Ned1_p = P_p^- Lambda^1 in the scaled Whitney-product basis
((p-1)!/alpha!) lambda^alpha w_ij with i<j, |alpha| = p-1, alpha_k = 0 for k < i
(DESIGN.md R-S1; rank pinned in tests); RT_p = P_p^- Lambda^2 in the
Whitney 2-form products ((p-1)!/alpha!) lambda^alpha w_ijk, i<j<k,
alpha_m = 0 for m < i. The span only affects rounding: the
dual basis is fixed by the dofs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .xprec import LD, eigh_ld, inv_ld, mm_ld, qr_pos_ld
from .simplex import (Simplex, canonical, reference_tet, multi_indices, mi_lookup,
                      TET_EDGES, TET_FACES, trace0, trace1, trace2, pairs)

ZERO_MODE_TOL = 1e-8      # R-A7: mu < 1e-8 max mu is kernel
CLUSTER_TOL = 1e-8        # R-A6: (mu_{j+1} - mu_j) <= 1e-8 mu_{j+1}
PROBE_ACCEPT = 1e-3       # R-A6 window acceptance
THETA = None


def _theta():
    s = lambda x: np.sqrt(LD(x))
    return np.array([s(2) - 1, s(3) - 1, s(5) - 2, s(7) - 2], dtype=LD)


def probe_bary(l: int, i: int) -> np.ndarray:
    """R-A6 probe point i (1-based) on an l-simplex: w_k = 1 + frac(i theta_k), normalised."""
    th = _theta()[: l + 1]
    x = LD(i) * th
    w = 1 + (x - np.floor(x))
    return (w / w.sum())[None, :]


def probe_dir(dim: int, i: int) -> np.ndarray:
    i = LD(i)
    if dim == 2:
        return np.array([np.cos(i), np.sin(i)], dtype=LD)
    if dim == 3:
        return np.array([np.sin(2 * i) * np.cos(i), np.sin(2 * i) * np.sin(i), np.cos(2 * i)], dtype=LD)
    raise ValueError


@dataclass
class Eigenbasis:
    """Canonicalized bubble eigenbasis on a canonical l-simplex."""
    l: int
    kind: str            # "cg" (0-forms, deg p) or "ned" (1-forms, deg p)
    lam: np.ndarray      # lambda_j = 1/mu_j, descending
    mu: np.ndarray
    F: np.ndarray        # rows: frame coefficients of psi_j (0-form deg p or 1-form deg p)
    n_kernel: int
    min_rel_gap: float = field(default=float("inf"))


def _canonicalize(S: Simplex, kind: str, mu, F, q):
    """R-A6: make psi unique inside eigenvalue clusters and fix signs."""
    n = len(mu)
    lam = 1 / mu
    j = 0
    F = F.copy()
    while j < n:
        c = 1
        while j + c < n and (mu[j + c] - mu[j + c - 1]) <= CLUSTER_TOL * mu[j + c]:
            c += 1
        blk = F[j:j + c]
        rho = np.max(np.sqrt(lam[j:j + c] / S.vol))
        s = 0
        while True:
            P = np.zeros((c, c), dtype=LD)
            for i in range(c):
                y = probe_bary(S.l, s + 1 + i)
                if kind == "cg":
                    P[i] = S.eval0(blk, q, y)[0]
                elif kind == "ned":
                    P[i] = S.eval1(blk, q, y)[0] @ probe_dir(S.dim, s + 1 + i)
                else:  # "rt": 2-form vector proxy in T-hat
                    P[i] = S.eval2(blk, q, y)[0] @ probe_dir(S.dim, s + 1 + i)
            smin = np.linalg.svd(P.astype(np.float64), compute_uv=False).min()
            if smin >= PROBE_ACCEPT * float(rho):
                break
            s += 1
            if s > 200:
                raise RuntimeError("probe window search failed")
        Q, R = qr_pos_ld(P.T)
        F[j:j + c] = Q.T @ blk
        j += c
    return F


def bubble_eigen(S: Simplex, kind: str, Fspan, q: int, dim_bubble: int, n_kernel: int) -> Eigenbasis:
    """Solve Eq. 3.9 on span(Fspan) (rows may be redundant), drop the kernel,
    renormalise to Eq. 3.8, canonicalize (R-A5, R-A6)."""
    if kind == "cg":
        M = S.mass0(Fspan, q, Fspan, q)
        dF = mm_ld(Fspan, S.grad_op(q))
        K = S.mass1(dF, q - 1, dF, q - 1)
    elif kind == "ned":
        M = S.mass1(Fspan, q, Fspan, q)
        dF = mm_ld(Fspan, S.curl_op(q))
        K = S.mass2(dF, q - 1, dF, q - 1)
    else:  # "rt": 2-forms on T-hat, d = div (Eq. 3.17)
        M = S.mass2(Fspan, q, Fspan, q)
        dF = mm_ld(Fspan, S.div_op(q))
        K = S.mass0(dF, q - 1, dF, q - 1)
    s, U = eigh_ld(M)
    keep = s > LD(1e-13) * s.max()
    assert int(keep.sum()) == dim_bubble, (kind, S.l, int(keep.sum()), dim_bubble)
    D = U[:, keep] / np.sqrt(s[keep])[None, :]
    Kp = mm_ld(mm_ld(D.T, K), D)
    mu, Y = eigh_ld(Kp)
    nz = mu > LD(ZERO_MODE_TOL) * mu.max()
    assert int((~nz).sum()) == n_kernel, (kind, S.l, int((~nz).sum()), n_kernel)
    mu = mu[nz]
    Fhat = mm_ld(mm_ld(D, Y[:, nz]).T, Fspan)         # M-orthonormal psi-hat
    F = Fhat / np.sqrt(mu)[:, None]          # Eq. 3.8 normalisation
    gaps = [(mu[k + 1] - mu[k]) / mu[k + 1] for k in range(len(mu) - 1)
            if (mu[k + 1] - mu[k]) > CLUSTER_TOL * mu[k + 1]]
    F = _canonicalize(S, kind, mu, F, q)
    return Eigenbasis(l=S.l, kind=kind, lam=1 / mu, mu=mu, F=F, n_kernel=n_kernel,
                      min_rel_gap=float(min(gaps)) if gaps else float("inf"))


@lru_cache(maxsize=None)
def cg_bubbles(l: int, p: int) -> Eigenbasis:
    """H(grad) bubble eigenbasis on the canonical l-simplex (Eq. 3.13):
    bubble space b_S P_{p-l-1} = span{lambda^alpha : |alpha|=p, alpha_k >= 1}."""
    S = canonical(l)
    A = multi_indices(l + 1, p)
    rows = np.nonzero(np.all(A >= 1, axis=1))[0]
    F = np.zeros((len(rows), len(A)), dtype=LD)
    F[np.arange(len(rows)), rows] = [_multinom(A[r]) for r in rows]
    dim = math.comb(p - 1, l)
    if dim == 0:
        return Eigenbasis(l=l, kind="cg", lam=np.zeros(0, LD), mu=np.zeros(0, LD),
                          F=np.zeros((0, len(A)), LD), n_kernel=0)
    return bubble_eigen(S, "cg", F, p, dim, 0)


def ned_bubble_span(l: int, p: int):
    """Whitney products lambda^alpha w_ij, |alpha| = p-1, i<j, with
    supp(alpha) U {i,j} = all vertices of the l-simplex (DESIGN.md R-S2)."""
    nv = l + 1
    out = []
    for (i, j) in pairs(nv):
        for a in multi_indices(nv, p - 1):
            cov = set(np.nonzero(a)[0]) | {i, j}
            if len(cov) == nv:
                out.append((tuple(a), i, j))
    return out


@lru_cache(maxsize=None)
def ned_bubbles(l: int, p: int) -> Eigenbasis:
    """Type-I Ned1 bubble eigenbasis on the canonical face (l=2) or cell (l=3),
    Eq. 3.15 via the augmented problem Eq. 3.9."""
    S = canonical(l)
    if l == 2:
        dim, nk = p * (p - 1), (p - 1) * (p - 2) // 2
    else:
        dim, nk = p * (p - 1) * (p - 2) // 2, (p - 1) * (p - 2) * (p - 3) // 6
    nv = l + 1
    if dim == 0:
        return Eigenbasis(l=l, kind="ned", lam=np.zeros(0, LD), mu=np.zeros(0, LD),
                          F=np.zeros((0, len(multi_indices(nv, p)) * nv), LD), n_kernel=0)
    elems = ned_bubble_span(l, p)
    F = S.whitney_products(elems, p - 1) * np.array([_multinom(a) for a, _, _ in elems], dtype=LD)[:, None]
    return bubble_eigen(S, "ned", F, p, dim, nk)


def rt_bubble_span(p: int):
    """Whitney 2-form products lambda^alpha w_ijk, |alpha| = p-1, i<j<k, with
    supp(alpha) U {i,j,k} = all four vertices of T-hat (the 2-form analogue of
    DESIGN.md R-S2)."""
    out = []
    for (i, j, k) in [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)]:
        for a in multi_indices(4, p - 1):
            if len(set(np.nonzero(a)[0]) | {i, j, k}) == 4:
                out.append((tuple(a), i, j, k))
    return out


@lru_cache(maxsize=None)
def rt_bubbles(p: int) -> Eigenbasis:
    """Type-I RT_p cell bubble eigenbasis Phi_{C,j} of Eq. 3.17:
    (div Phi_j, div Phi_i) = delta_ij, (Phi_j, Phi_i) = lambda_j delta_ij, via
    the augmented problem Eq. 3.9 on the whole bubble space, whose kernel (the
    divergence-free bubbles) has dimension dim RT-bubbles - (dim P_{p-1} - 1)."""
    T = reference_tet()
    dim = p * (p + 1) * (p - 1) // 2
    nI = p * (p + 1) * (p + 2) // 6 - 1
    npair = 6
    if dim == 0 or nI == 0:
        return Eigenbasis(l=3, kind="rt", lam=np.zeros(0, LD), mu=np.zeros(0, LD),
                          F=np.zeros((0, len(multi_indices(4, p)) * npair), LD), n_kernel=dim)
    elems = rt_bubble_span(p)
    F = T.whitney2_products(elems, p - 1) * np.array([_multinom(a) for a, _, _, _ in elems], dtype=LD)[:, None]
    return bubble_eigen(T, "rt", F, p, dim, dim - nI)


# ------------------------------------------------------------------ elements
@dataclass
class RefElement:
    space: str                 # "hgrad" | "hcurl"
    p: int
    n: int
    T: Simplex
    span: np.ndarray           # rows = basis fields of the span (0-form or 1-form, deg p)
    C: np.ndarray              # phi_j = sum_k C[k, j] span_k  (longdouble)
    dof_entity: list           # per local dof: (dim, local entity index, j, type)
    V: np.ndarray              # Vandermonde l_i(span_j)
    lam_cell: np.ndarray       # cell eigenvalues (type-I)

    @property
    def interior(self):
        return np.array([e[0] == 3 for e in self.dof_entity])


def _multinom(a) -> int:
    out = math.factorial(int(sum(a)))
    for x in a:
        out //= math.factorial(int(x))
    return out


def _entity_lists():
    return [(0, [(i,) for i in range(4)]), (1, TET_EDGES), (2, TET_FACES), (3, [(0, 1, 2, 3)])]


@lru_cache(maxsize=None)
def cg_element(p: int) -> RefElement:
    """CG_p with the dofs of Eq. 3.14: vertex values, then
    (grad_S psi_{S,j}, grad_S v)_S on edges, faces and the cell."""
    T = reference_tet()
    A = multi_indices(4, p)
    n = len(A)
    # scaled Bernstein basis (p!/beta!) lambda^beta (R-S1)
    B = np.diag(np.array([_multinom(a) for a in A], dtype=LD))
    lk = mi_lookup(4, p)
    rows, ents = [], []
    for dim, ents_d in _entity_lists():
        for ei, s in enumerate(ents_d):
            if dim == 0:
                e = [0, 0, 0, 0]
                e[s[0]] = p
                rows.append(B[:, lk[tuple(e)]].copy())  # v(V_i): lambda^gamma(V_i) = [gamma = p e_i]
                ents.append((0, ei, 0, "I"))
                continue
            eb = cg_bubbles(dim, p)
            if len(eb.lam) == 0:
                continue
            Sc = canonical(dim) if dim < 3 else T
            tr = trace0(B, p, 4, s) if dim < 3 else B
            g_psi = mm_ld(eb.F, Sc.grad_op(p))
            g_v = mm_ld(tr, Sc.grad_op(p))
            Vs = Sc.mass1(g_psi, p - 1, g_v, p - 1)
            for j in range(len(eb.lam)):
                rows.append(Vs[j])
                ents.append((dim, ei, j, "I"))
    V = np.array(rows, dtype=LD)
    assert V.shape == (n, n)
    C = inv_ld(V)
    return RefElement("hgrad", p, n, T, B, C, ents, V, cg_bubbles(3, p).lam)


def ned_span(p: int):
    """Whitney-product basis of Ned1_p(T-hat): lambda^alpha w_ij, i<j, |alpha|=p-1,
    alpha_k = 0 for k < i (DESIGN.md R-S1)."""
    out = []
    for (i, j) in pairs(4):
        for a in multi_indices(4, p - 1):
            if all(a[k] == 0 for k in range(i)):
                out.append((tuple(a), i, j))
    return out


@lru_cache(maxsize=None)
def ned_element(p: int) -> RefElement:
    """Ned1_p with the dofs of Eq. 3.16, ordered per entity:
    edge: Whitney (1, t.v)_E then type-II (grad_E psi_{E,j}, t.v)_E;
    face / cell: type-I (curl Psi_j, curl v) then type-II (grad psi_j, v)."""
    T = reference_tet()
    elems = ned_span(p)
    # scaled Whitney products ((p-1)!/alpha!) lambda^alpha w_ij (R-S1)
    Fb = T.whitney_products(elems, p - 1) * np.array([_multinom(a) for a, _, _ in elems], dtype=LD)[:, None]
    n = len(elems)
    rows, ents = [], []
    for dim, ents_d in _entity_lists():
        if dim == 0:
            continue
        for ei, s in enumerate(ents_d):
            Sc = canonical(dim) if dim < 3 else T
            tr = trace1(Fb, p, 4, s) if dim < 3 else Fb
            if dim == 1:
                # Whitney: (1, t.v)_E with t = g_1 - g_0 = unit tangent from lower to higher vertex
                t = np.zeros((1, 2), dtype=LD)
                t[0, 0], t[0, 1] = -1, 1
                rows.append(Sc.mass1(t, 0, tr, p)[0])
                ents.append((1, ei, 0, "W"))
            else:
                Psi = ned_bubbles(dim, p)
                if len(Psi.lam):
                    cP = mm_ld(Psi.F, Sc.curl_op(p))
                    cv = mm_ld(tr, Sc.curl_op(p))
                    Vs = Sc.mass2(cP, p - 1, cv, p - 1)
                    for j in range(len(Psi.lam)):
                        rows.append(Vs[j])
                        ents.append((dim, ei, j, "I"))
            psi = cg_bubbles(dim, p)
            if len(psi.lam):
                g_psi = mm_ld(psi.F, Sc.grad_op(p))
                Vs = Sc.mass1(g_psi, p - 1, tr, p)
                for j in range(len(psi.lam)):
                    rows.append(Vs[j])
                    ents.append((dim, ei, j, "II"))
    V = np.array(rows, dtype=LD)
    assert V.shape == (n, n), V.shape
    C = inv_ld(V)
    return RefElement("hcurl", p, n, T, Fb, C, ents, V, ned_bubbles(3, p).lam)


def rt_span(p: int):
    """Whitney 2-form product basis of RT_p(T-hat) = P_p^- Lambda^2:
    lambda^alpha w_ijk, i<j<k, |alpha| = p-1, alpha_m = 0 for m < i (the 2-form
    analogue of DESIGN.md R-S1; dimension p(p+1)(p+3)/2, asserted)."""
    out = []
    for (i, j, k) in [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)]:
        for a in multi_indices(4, p - 1):
            if all(a[m] == 0 for m in range(i)):
                out.append((tuple(a), i, j, k))
    assert len(out) == p * (p + 1) * (p + 3) // 2
    return out


def face_unit_form(F: Simplex) -> np.ndarray:
    """The constant 2-form on the canonical face whose proxy is 1 (orientation
    c0 -> c1 -> c2, i.e. the sorted vertex order, DESIGN.md R-D2): c g_0 x g_1
    with c = 1 / (g_0 x g_1)."""
    cr = F.g[0][0] * F.g[1][1] - F.g[0][1] * F.g[1][0]
    u = np.zeros((1, 3), dtype=LD)
    u[0, 0] = 1 / cr          # pair (0,1) is the first of the face's pair frame
    return u


@lru_cache(maxsize=None)
def rt_element(p: int) -> RefElement:
    """RT_p with the dofs of Eq. 3.18, ordered per entity:
    face: Whitney (1, n.v)_F then type-II (curl_F Psi_{F,j}, n.v)_F;
    cell: type-I (div Phi_{C,j}, div v) then type-II (curl Psi_{C,j}, v).
    Psi are the Ned1_p bubble eigenbases (DESIGN.md R-D1: the paper allows
    Ned1_p or Ned2_p here)."""
    T = reference_tet()
    elems = rt_span(p)
    Fb = T.whitney2_products(elems, p - 1) * np.array([_multinom(a) for a, _, _, _ in elems], dtype=LD)[:, None]
    n = len(elems)
    rows, ents = [], []
    Sc = canonical(2)
    u = face_unit_form(Sc)
    PsiF = ned_bubbles(2, p)
    cPsiF = mm_ld(PsiF.F, Sc.curl_op(p)) if len(PsiF.lam) else None
    for ei, s in enumerate(TET_FACES):
        tr = trace2(Fb, p, 4, s)
        rows.append(Sc.mass2(u, 0, tr, p)[0])
        ents.append((2, ei, 0, "W"))
        if cPsiF is not None:
            Vs = Sc.mass2(cPsiF, p - 1, tr, p)
            for j in range(len(PsiF.lam)):
                rows.append(Vs[j])
                ents.append((2, ei, j, "II"))
    Phi = rt_bubbles(p)
    if len(Phi.lam):
        Vs = T.mass0(mm_ld(Phi.F, T.div_op(p)), p - 1, mm_ld(Fb, T.div_op(p)), p - 1)
        for j in range(len(Phi.lam)):
            rows.append(Vs[j])
            ents.append((3, 0, j, "I"))
    PsiC = ned_bubbles(3, p)
    if len(PsiC.lam):
        Vs = T.mass2(mm_ld(PsiC.F, T.curl_op(p)), p - 1, Fb, p)
        for j in range(len(PsiC.lam)):
            rows.append(Vs[j])
            ents.append((3, 0, j, "II"))
    V = np.array(rows, dtype=LD)
    assert V.shape == (n, n), V.shape
    C = inv_ld(V)
    return RefElement("hdiv", p, n, T, Fb, C, ents, V, Phi.lam)


def element(space: str, p: int) -> RefElement:
    return {"hgrad": cg_element, "hcurl": ned_element, "hdiv": rt_element}[space](p)


# ------------------------------------------------------------------ tabulation
def tabulate(el: RefElement, bary):
    """Values and exterior derivatives of the reference basis at barycentric
    points of T-hat, Cartesian components, in longdouble.
    hgrad: (phi [npts,n], grad [npts,n,3]); hcurl: (phi [npts,n,3], curl [npts,n,3])."""
    T, p = el.T, el.p
    if el.space == "hgrad":
        Phi = mm_ld(el.C.T, el.span)  # rows = phi_j in monomial coefficients
        val = T.eval0(Phi, p, bary)
        der = T.eval1(mm_ld(Phi, T.grad_op(p)), p - 1, bary)
        return val, der
    Phi = mm_ld(el.C.T, el.span)
    if el.space == "hdiv":  # (phi [npts,n,3] 2-form proxies, div [npts,n])
        return T.eval2(Phi, p, bary), T.eval0(mm_ld(Phi, T.div_op(p)), p - 1, bary)
    val = T.eval1(Phi, p, bary)
    der = T.eval2(mm_ld(Phi, T.curl_op(p)), p - 1, bary)
    return val, der


def reference_matrices(el: RefElement):
    """M-hat and K-hat^{ab} (Cartesian a,b) by exact integration, longdouble.
    hgrad: M [n,n], K [3,3,n,n] with K^{ab}_ij = int d_a phi_i d_b phi_j.
    hcurl: M [3,3,n,n] with M^{ab}_ij = int phi_i,a phi_j,b; K likewise with curls.
    hdiv: M [3,3,n,n] of the 2-form proxies; K [n,n] with divergences."""
    T, p, C = el.T, el.p, el.C
    if el.space == "hgrad":
        Mh = mm_ld(mm_ld(C.T, T.mass0(el.span, p, el.span, p)), C)
        G = mm_ld(el.span, T.grad_op(p))
        Np1 = len(multi_indices(4, p - 1))
        Gr = G.reshape(el.n, Np1, 4)
        Dc = [mm_ld(C.T, Gr @ T.g[:, a]) for a in range(3)]
        I1 = T.I(p - 1, p - 1)
        K = np.array([[mm_ld(mm_ld(Dc[a], I1), Dc[b].T) for b in range(3)] for a in range(3)])
        return Mh, K
    Np = len(multi_indices(4, p))
    if el.space == "hdiv":  # M^{ab}_ij = int phi_i,a phi_j,b (2-form proxies), K_ij = int div phi_i div phi_j
        cr = np.array([np.cross(T.g[a], T.g[b]) for a, b in T.pairs], dtype=LD)
        Pr = el.span.reshape(el.n, Np, len(T.pairs))
        Pc = [mm_ld(C.T, Pr @ cr[:, a]) for a in range(3)]
        Ip = T.I(p, p)
        M = np.array([[mm_ld(mm_ld(Pc[a], Ip), Pc[b].T) for b in range(3)] for a in range(3)])
        Dv = mm_ld(C.T, mm_ld(el.span, T.div_op(p)))
        return M, mm_ld(mm_ld(Dv, T.I(p - 1, p - 1)), Dv.T)
    Pr = el.span.reshape(el.n, Np, 4)
    Pc = [mm_ld(C.T, Pr @ T.g[:, a]) for a in range(3)]
    Ip = T.I(p, p)
    M = np.array([[mm_ld(mm_ld(Pc[a], Ip), Pc[b].T) for b in range(3)] for a in range(3)])
    cr = np.array([np.cross(T.g[a], T.g[b]) for a, b in T.pairs], dtype=LD)
    Np1 = len(multi_indices(4, p - 1))
    Cf = mm_ld(el.span, T.curl_op(p)).reshape(el.n, Np1, len(T.pairs))
    Rc = [mm_ld(C.T, Cf @ cr[:, a]) for a in range(3)]
    I1 = T.I(p - 1, p - 1)
    K = np.array([[mm_ld(mm_ld(Rc[a], I1), Rc[b].T) for b in range(3)] for a in range(3)])
    return M, K
