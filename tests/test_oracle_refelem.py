"""Pins for the oracle's reference elements (oracle/simplex.py, oracle/refelem.py).

Each check is pinned to something other than the code it checks: closed forms
(textbook simplex integrals, hand-derived eigenvalues), the paper's lemmas
(P:906-1229), or re-integration with an independent quadrature rule.
"""
import math

import numpy as np
import pytest
from numpy.polynomial.legendre import leggauss

from oracle.xprec import LD
from oracle.simplex import canonical, reference_tet, multi_indices, TET_EDGES, TET_FACES
from oracle.refelem import (cg_bubbles, ned_bubbles, cg_element, ned_element, reference_matrices,
                            tabulate, ned_span)
from oracle.fem import tet_quadrature, gauss_jacobi01


# ------------------------------------------------------------------ geometry
def test_reference_geometry_closed_forms():
    """R-A1: edge length 2; grad(lambda).grad(lambda) = 1/4,-1/4 (edge), 1/3,-1/6 (face),
    3/8,-1/8 (tet); volumes 2, sqrt3, 2 sqrt2 / 3."""
    for l, (d, o, vol) in {1: (1 / 4, -1 / 4, 2.0), 2: (1 / 3, -1 / 6, math.sqrt(3)),
                           3: (3 / 8, -1 / 8, 2 * math.sqrt(2) / 3)}.items():
        S = canonical(l)
        G = S.G.astype(float)
        assert np.allclose(np.diag(G), d, rtol=0, atol=1e-15)
        assert np.allclose(G[~np.eye(l + 1, dtype=bool)], o, rtol=0, atol=1e-15)
        assert abs(float(S.vol) - vol) < 1e-15
        c = S.coords.astype(float)
        for a in range(l + 1):
            for b in range(a + 1, l + 1):
                assert abs(np.linalg.norm(c[a] - c[b]) - 2) < 1e-15
    assert np.allclose(reference_tet().coords.astype(float).mean(axis=0), 0, atol=1e-15)


def test_exact_simplex_integrals_against_quadrature():
    """int_T lambda^a = 3! |T| a! / (|a|+3)! vs the conical product rule (textbook)."""
    T = reference_tet()
    lam, w = tet_quadrature(10)
    for q in range(0, 11):
        A = multi_indices(4, q)
        vals = w @ np.prod(lam[:, None, :] ** A[None], axis=2) * float(T.vol)
        ex = T.I(q, 0)[:, 0].astype(float)
        assert np.allclose(vals, ex, rtol=1e-13, atol=0)
        # closed form by hand
        for a, v in zip(A, ex):
            cf = 6 * float(T.vol) * np.prod([math.factorial(x) for x in a]) / math.factorial(q + 3)
            assert abs(v - cf) <= 1e-14 * cf


# ------------------------------------------------------------------ eigenvalues
@pytest.mark.parametrize("p,lams", [
    (2, [2 / 5]), (3, [2 / 5, 2 / 21]),
    (4, [0.405278771343981, 2 / 21, 0.0391656731004637]),
    (5, [0.405278771343981, 0.10126184201514761, 0.0391656731004637, 0.019950279196973467]),
])
def test_cg_edge_eigenvalues(p, lams):
    """SPEC S:155-156 / SURVEY F4: closed forms of the edge bubble problem (length 2)."""
    got = cg_bubbles(1, p).lam.astype(float)
    assert np.allclose(got, lams, rtol=1e-12, atol=0)


def test_cg_face_cell_eigenvalues():
    assert abs(float(cg_bubbles(2, 3).lam[0]) - 1 / 14) < 1e-15
    assert abs(float(cg_bubbles(3, 4).lam[0]) - 4 / 165) < 1e-16


def test_cg_high_p_eigenvalues():
    """SURVEY F9 (40-digit exact-rational + mpmath computation)."""
    f12 = cg_bubbles(2, 12).lam.astype(float)
    assert abs(f12[0] / 0.075990887731724982 - 1) < 1e-13
    assert abs(f12[1] / 0.032567523228218717 - 1) < 1e-13
    c10 = cg_bubbles(3, 10).lam.astype(float)
    assert abs(c10[0] / 0.026494830338735314 - 1) < 1e-13
    assert abs(c10[1] / 0.014350135244637459 - 1) < 1e-13


def test_ned_eigenvalues():
    """SURVEY F5 (8-digit values; degenerate clusters are exact)."""
    f2 = ned_bubbles(2, 2).lam.astype(float)
    assert np.allclose(f2, [2 / 9, 2 / 9], rtol=1e-14)
    f3 = ned_bubbles(2, 3).lam.astype(float)
    assert np.allclose(f3, [0.22724752, 0.22724752, 1 / 14, 0.05301041, 0.05301041], rtol=1e-8)
    c3 = ned_bubbles(3, 3).lam.astype(float)
    assert np.allclose(c3, [7 / 144] * 3, rtol=1e-14)
    c4 = ned_bubbles(3, 4).lam.astype(float)
    ref = [0.04877649] * 3 + [1 / 45] * 3 + [2 / 99] * 2 + [0.01921774] * 3
    assert np.allclose(c4, ref, rtol=1e-8)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_dimensions_and_kernel_counts(p):
    """Eq. 3.7 bookkeeping; kernel of Eq. 3.9 = N^{k-1}_S."""
    for l in (1, 2, 3):
        assert len(cg_bubbles(l, p).lam) == math.comb(p - 1, l)
    assert len(ned_bubbles(2, p).lam) == (p - 1) * (p + 2) // 2
    assert ned_bubbles(2, p).n_kernel == (p - 1) * (p - 2) // 2
    assert len(ned_bubbles(3, p).lam) == (p - 1) * (p - 2) * (2 * p + 3) // 6
    assert ned_bubbles(3, p).n_kernel == (p - 1) * (p - 2) * (p - 3) // 6
    assert cg_element(p).n == (p + 1) * (p + 2) * (p + 3) // 6
    assert ned_element(p).n == p * (p + 2) * (p + 3) // 2
    if p == 4:
        assert len(ned_bubbles(2, 4).lam) == 9
        ents = [e[0] for e in cg_element(4).dof_entity]
        assert [ents.count(d) for d in range(4)] == [4, 18, 12, 1]


# ------------------------------------------------------------------ quadrature rules for re-integration
def edge_rule(m):
    x, w = leggauss(m)
    bary = np.stack([(1 - x) / 2, (1 + x) / 2], axis=1)
    return bary, w  # ds = dx on the length-2 edge


def tri_rule(m):
    u, wu = gauss_jacobi01(m, 1.0)
    v, wv = gauss_jacobi01(m, 0.0)
    U, V = np.meshgrid(u, v, indexing="ij")
    W = wu[:, None] * wv[None, :]
    xi, eta = U, (1 - U) * V
    bary = np.stack([1 - xi - eta, xi, eta], axis=-1).reshape(-1, 3)
    return bary, W.reshape(-1) * 2.0 * math.sqrt(3)  # weights sum to |F| = sqrt 3


def rule(l, m):
    if l == 1:
        return edge_rule(m)
    if l == 2:
        return tri_rule(m)
    lam, w = tet_quadrature(2 * m - 1)
    return lam, w * float(reference_tet().vol)


@pytest.mark.parametrize("p", [3, 5, 7])
def test_cg_eigen_orthogonality_by_quadrature(p):
    """Eq. 3.8: (grad psi_i, grad psi_j) = delta_ij, (psi_i, psi_j) = lambda_j delta_ij,
    re-integrated with a Gauss rule."""
    for l in (1, 2, 3):
        eb = cg_bubbles(l, p)
        if not len(eb.lam):
            continue
        S = canonical(l)
        bary, w = rule(l, p + 2)
        bary = bary.astype(LD)
        v = S.eval0(eb.F, p, bary).astype(float)
        g = S.eval1(eb.F @ S.grad_op(p), p - 1, bary).astype(float)
        M = np.einsum("q,qi,qj->ij", w, v, v)
        K = np.einsum("q,qid,qjd->ij", w, g, g)
        assert np.allclose(K, np.eye(len(eb.lam)), atol=1e-12)
        assert np.allclose(M, np.diag(eb.lam.astype(float)), atol=1e-13)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_ned_eigen_orthogonality_by_quadrature(p):
    """Eq. 3.15: (curl Psi_i, curl Psi_j) = delta_ij, (Psi_i, Psi_j) = lambda_j delta_ij;
    type-I Psi are L2-orthogonal to the gradients of the CG bubbles (Eq. 3.4)."""
    for l in (2, 3):
        eb = ned_bubbles(l, p)
        if not len(eb.lam):
            continue
        S = canonical(l)
        bary, w = rule(l, p + 2)
        bary = bary.astype(LD)
        v = S.eval1(eb.F, p, bary).astype(float)
        c = S.eval2(eb.F @ S.curl_op(p), p - 1, bary).astype(float)
        M = np.einsum("q,qid,qjd->ij", w, v, v)
        if l == 2:
            K = np.einsum("q,qi,qj->ij", w, c, c)
        else:
            K = np.einsum("q,qid,qjd->ij", w, c, c)
        assert np.allclose(K, np.eye(len(eb.lam)), atol=1e-12)
        assert np.allclose(M, np.diag(eb.lam.astype(float)), atol=1e-13)
        cb = cg_bubbles(l, p)
        if len(cb.lam):
            g = S.eval1(cb.F @ S.grad_op(p), p - 1, bary).astype(float)
            assert np.abs(np.einsum("q,qid,qjd->ij", w, v, g)).max() < 1e-13


def test_canonicalization_rule():
    """R-A6: inside each eigenvalue cluster, probe_i(psi_j) is lower triangular with
    positive diagonal (checked on the Ned1 face p=3 pairs and the cell p=4 triples)."""
    from oracle.refelem import probe_bary, probe_dir
    for (l, p) in ((2, 3), (3, 4), (3, 3)):
        eb = ned_bubbles(l, p)
        S = canonical(l)
        mu = eb.mu.astype(float)
        j = 0
        while j < len(mu):
            c = 1
            while j + c < len(mu) and mu[j + c] - mu[j + c - 1] <= 1e-8 * mu[j + c]:
                c += 1
            if c > 1:
                # the accepted window starts at s = 0 for these cases
                P = np.array([[float(S.eval1(eb.F[j + k:j + k + 1], p, probe_bary(l, i + 1))[0, 0]
                                     @ probe_dir(l, i + 1)) for k in range(c)] for i in range(c)])
                assert np.all(np.diag(P) > 0)
                assert np.abs(np.triu(P, 1)).max() < 1e-14
            j += c


# ------------------------------------------------------------------ dofs by quadrature
def _edge_points(a, b, m):
    bary_e, w = edge_rule(m)
    bary = np.zeros((len(w), 4))
    bary[:, a], bary[:, b] = bary_e[:, 0], bary_e[:, 1]
    return bary_e, bary, w


def _face_frame(f):
    T = reference_tet()
    Vh = T.coords.astype(float)
    Fc = canonical(2).coords.astype(float)
    Q = np.column_stack([Vh[f[1]] - Vh[f[0]], Vh[f[2]] - Vh[f[0]]]) @ np.linalg.inv(
        np.column_stack([Fc[1] - Fc[0], Fc[2] - Fc[0]]))
    return Q


@pytest.mark.parametrize("p", [3, 4])
def test_cg_duality_by_quadrature(p):
    """l_i(phi_j) = delta_ij, each dof of Eq. 3.14 re-evaluated by quadrature."""
    el = cg_element(p)
    E1 = canonical(1)
    F2 = canonical(2)
    T = reference_tet()
    rows = []
    for (dim, ei, j, typ) in el.dof_entity:
        if dim == 0:
            bary = np.zeros((1, 4))
            bary[0, ei] = 1
            rows.append(tabulate(el, bary.astype(LD))[0].astype(float)[0])
        elif dim == 1:
            a, b = TET_EDGES[ei]
            be, bary, w = _edge_points(a, b, p + 2)
            t = (T.coords[b] - T.coords[a]).astype(float) / 2
            psi = cg_bubbles(1, p)
            dpsi = E1.eval1(psi.F[j:j + 1] @ E1.grad_op(p), p - 1, be.astype(LD)).astype(float)[:, 0, 0]
            g = tabulate(el, bary.astype(LD))[1].astype(float)
            rows.append(np.einsum("q,q,qn->n", w, dpsi, g @ t))
        elif dim == 2:
            f = TET_FACES[ei]
            bf, wf = tri_rule(p + 2)
            bary = np.zeros((len(wf), 4))
            bary[:, list(f)] = bf
            Q = _face_frame(f)
            psi = cg_bubbles(2, p)
            dpsi = F2.eval1(psi.F[j:j + 1] @ F2.grad_op(p), p - 1, bf.astype(LD)).astype(float)[:, 0, :] @ Q.T
            g = tabulate(el, bary.astype(LD))[1].astype(float)
            rows.append(np.einsum("q,qd,qnd->n", wf, dpsi, g))
        else:
            lam, w = tet_quadrature(2 * p)
            w = w * float(T.vol)
            psi = cg_bubbles(3, p)
            dpsi = T.eval1(psi.F[j:j + 1] @ T.grad_op(p), p - 1, lam.astype(LD)).astype(float)[:, 0, :]
            g = tabulate(el, lam.astype(LD))[1].astype(float)
            rows.append(np.einsum("q,qd,qnd->n", w, dpsi, g))
    D = np.array(rows)
    assert np.abs(D - np.eye(el.n)).max() < 1e-11


@pytest.mark.parametrize("p", [2, 3, 4])
def test_ned_duality_by_quadrature(p):
    """l_i(phi_j) = delta_ij for the dofs of Eq. 3.16, re-evaluated by quadrature."""
    el = ned_element(p)
    E1, F2, T = canonical(1), canonical(2), reference_tet()
    rows = []
    for (dim, ei, j, typ) in el.dof_entity:
        if dim == 1:
            a, b = TET_EDGES[ei]
            be, bary, w = _edge_points(a, b, p + 2)
            t = (T.coords[b] - T.coords[a]).astype(float) / 2
            phi = tabulate(el, bary.astype(LD))[0].astype(float)
            tphi = phi @ t
            if typ == "W":
                rows.append(w @ tphi)
            else:
                psi = cg_bubbles(1, p)
                dpsi = E1.eval1(psi.F[j:j + 1] @ E1.grad_op(p), p - 1, be.astype(LD)).astype(float)[:, 0, 0]
                rows.append(np.einsum("q,q,qn->n", w, dpsi, tphi))
        elif dim == 2:
            f = TET_FACES[ei]
            bf, wf = tri_rule(p + 2)
            bary = np.zeros((len(wf), 4))
            bary[:, list(f)] = bf
            Q = _face_frame(f)
            nrm = np.cross(Q[:, 0], Q[:, 1])
            phi, cphi = [x.astype(float) for x in tabulate(el, bary.astype(LD))]
            if typ == "I":
                Psi = ned_bubbles(2, p)
                cP = F2.eval2(Psi.F[j:j + 1] @ F2.curl_op(p), p - 1, bf.astype(LD)).astype(float)[:, 0]
                rows.append(np.einsum("q,q,qn->n", wf, cP, cphi @ nrm))
            else:
                psi = cg_bubbles(2, p)
                dpsi = F2.eval1(psi.F[j:j + 1] @ F2.grad_op(p), p - 1, bf.astype(LD)).astype(float)[:, 0, :] @ Q.T
                rows.append(np.einsum("q,qd,qnd->n", wf, dpsi, phi))
        else:
            lam, w = tet_quadrature(2 * p)
            w = w * float(T.vol)
            phi, cphi = [x.astype(float) for x in tabulate(el, lam.astype(LD))]
            if typ == "I":
                Psi = ned_bubbles(3, p)
                cP = T.eval2(Psi.F[j:j + 1] @ T.curl_op(p), p - 1, lam.astype(LD)).astype(float)[:, 0, :]
                rows.append(np.einsum("q,qd,qnd->n", w, cP, cphi))
            else:
                psi = cg_bubbles(3, p)
                dpsi = T.eval1(psi.F[j:j + 1] @ T.grad_op(p), p - 1, lam.astype(LD)).astype(float)[:, 0, :]
                rows.append(np.einsum("q,qd,qnd->n", w, dpsi, phi))
    D = np.array(rows)
    assert np.abs(D - np.eye(el.n)).max() < 1e-11


# ------------------------------------------------------------------ lemmas
def _random_bary(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.dirichlet(np.ones(4), n)
    return x


@pytest.mark.parametrize("p", [1, 3, 5])
def test_lemma41_whitney_containment(p):
    """Lemma 4.1: vertex functions = barycentrics; Ned1 edge Whitney
    functions = lambda_a grad lambda_b - lambda_b grad lambda_a."""
    bary = _random_bary(50, p)
    T = reference_tet()
    g = T.g.astype(float)
    el = cg_element(p)
    val = tabulate(el, bary.astype(LD))[0].astype(float)
    for i in range(4):
        assert np.abs(val[:, i] - bary[:, i]).max() < 1e-12
    el = ned_element(p)
    val = tabulate(el, bary.astype(LD))[0].astype(float)
    for k, (dim, ei, j, typ) in enumerate(el.dof_entity):
        if typ == "W":
            a, b = TET_EDGES[ei]
            w = bary[:, a:a + 1] * g[b] - bary[:, b:b + 1] * g[a]
            assert np.abs(val[:, k] - w).max() < 1e-12


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_lemma43_type2_is_gradient(p):
    """Lemma 4.3: phi^{1,II}_{S,n} = grad phi^{0,I}_{S,n}."""
    bary = _random_bary(40, 10 + p)
    cg, ned = cg_element(p), ned_element(p)
    gcg = tabulate(cg, bary.astype(LD))[1].astype(float)
    vn = tabulate(ned, bary.astype(LD))[0].astype(float)
    cg_index = {(d, e, j): k for k, (d, e, j, t) in enumerate(cg.dof_entity)}
    n = 0
    for k, (dim, ei, j, typ) in enumerate(ned.dof_entity):
        if typ == "II":
            assert np.abs(vn[:, k] - gcg[:, cg_index[(dim, ei, j)]]).max() < 1e-11
            n += 1
    assert n == sum(math.comb(p - 1, l) * c for l, c in ((1, 6), (2, 4), (3, 1)))


@pytest.mark.parametrize("p", [2, 4])
def test_lemma42_traces_are_eigenfunctions(p):
    """Lemma 4.2: tr_S phi_{S,j} = psi_{S,j}; functions of other
    entities of the same or higher dimension have zero trace on S."""
    el = cg_element(p)
    E1 = canonical(1)
    for ei, (a, b) in enumerate(TET_EDGES):
        be, bary, w = _edge_points(a, b, 5)
        val = tabulate(el, bary.astype(LD))[0].astype(float)
        psi = E1.eval0(cg_bubbles(1, p).F, p, be.astype(LD)).astype(float)
        for k, (dim, e2, j, typ) in enumerate(el.dof_entity):
            if dim == 1 and e2 == ei:
                assert np.abs(val[:, k] - psi[:, j]).max() < 1e-11
            elif dim >= 1:
                assert np.abs(val[:, k]).max() < 1e-11


@pytest.mark.parametrize("space,p", [("hgrad", 4), ("hgrad", 5), ("hgrad", 7), ("hcurl", 3), ("hcurl", 4), ("hcurl", 5)])
def test_lemma44_block_structure(space, p):
    """Lemma 4.4: K_IG = 0, K_II^{I,I} = I, M_II^{I,I} = Lambda,
    M_II^{II,II} = I, M_IG^{II,*} = 0, type-II rows of K vanish."""
    el = cg_element(p) if space == "hgrad" else ned_element(p)
    M, K = reference_matrices(el)
    if space == "hgrad":
        Mt, Kt = M.astype(float), sum(K[a, a] for a in range(3)).astype(float)
    else:
        Mt = sum(M[a, a] for a in range(3)).astype(float)
        Kt = sum(K[a, a] for a in range(3)).astype(float)
    I = el.interior
    typ = np.array([e[3] for e in el.dof_entity])
    II1 = I & (typ == "I")
    assert np.abs(Kt[np.ix_(I, ~I)]).max() < 1e-11
    assert np.abs(Kt[np.ix_(II1, II1)] - np.eye(II1.sum())).max() < 1e-11
    assert np.abs(Mt[np.ix_(II1, II1)] - np.diag(el.lam_cell.astype(float))).max() < 1e-11
    if space == "hcurl":
        II2 = I & (typ == "II")
        if II2.any():
            assert np.abs(Mt[np.ix_(II2, II2)] - np.eye(II2.sum())).max() < 1e-11
            assert np.abs(Mt[np.ix_(II2, ~I)]).max() < 1e-11
            assert np.abs(Mt[np.ix_(II2, II1)]).max() < 1e-11
        assert np.abs(Kt[typ == "II"]).max() < 1e-11


@pytest.mark.parametrize("p", [4, 6, 8])
def test_fig4_interior_conditioning(p):
    """Fig. 4: diagonally scaled interior M and K blocks have kappa = 1."""
    el = cg_element(p)
    M, K = reference_matrices(el)
    Kt = sum(K[a, a] for a in range(3)).astype(float)
    I = el.interior
    for B in (M.astype(float)[np.ix_(I, I)], Kt[np.ix_(I, I)]):
        d = 1 / np.sqrt(np.diag(B))
        assert abs(np.linalg.cond(d[:, None] * B * d[None, :]) - 1) < 1e-8


@pytest.mark.parametrize("space,p", [("hgrad", 5), ("hcurl", 4)])
def test_thmA1_pythagorean(space, p):
    """Thm A.1: ||du||^2 = ||du_Gamma||^2 + ||du_I||^2 on T-hat."""
    el = cg_element(p) if space == "hgrad" else ned_element(p)
    M, K = reference_matrices(el)
    Kt = sum(K[a, a] for a in range(3)).astype(float)
    rng = np.random.default_rng(5)
    I = el.interior
    for _ in range(5):
        u = rng.standard_normal(el.n)
        uI, uG = u * I, u * ~I
        tot = u @ Kt @ u
        assert abs(tot - (uG @ Kt @ uG + uI @ Kt @ uI)) < 1e-10 * tot


@pytest.mark.parametrize("p", [2, 3, 4])
def test_ned_span_is_first_kind(p):
    """Ned1_p = P_{p-1}^3 + P~_{p-1}^3 x x. The Whitney-product basis
    (R-S1) reproduces both parts exactly and has dimension p(p+2)(p+3)/2."""
    T = reference_tet()
    el = ned_element(p)
    bary = _random_bary(4 * el.n, 99).astype(LD)
    X = T.cart(bary).astype(float)
    vals = tabulate(el, bary)[0].astype(float)         # [npts, n, 3]
    B = vals.transpose(0, 2, 1).reshape(-1, el.n)
    assert np.linalg.matrix_rank(B, tol=1e-10 * np.abs(B).max()) == el.n == p * (p + 2) * (p + 3) // 2
    rng = np.random.default_rng(7)
    for trial in range(6):
        c = rng.standard_normal((3, len(multi_indices(4, p - 1))))
        mon = np.prod(np.c_[X, np.ones(len(X))][:, None, :] ** multi_indices(4, p - 1)[None], axis=2)
        q = mon @ c.T                                   # P_{p-1}^3 field
        if trial % 2:
            hom = np.prod(X[:, None, :] ** multi_indices(3, p - 1)[None], axis=2)
            qh = hom @ rng.standard_normal((3, hom.shape[1])).T
            q = np.cross(qh, X)                         # homogeneous part x x
        coef, res, rk, sv = np.linalg.lstsq(B, q.reshape(-1), rcond=None)
        assert np.abs(B @ coef - q.reshape(-1)).max() < 1e-9 * np.abs(q).max()
