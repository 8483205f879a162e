"""Pins for the oracle's global operator, preconditioner and PCG (oracle/mesh.py,
oracle/fem.py, oracle/solver.py) against textbook FEM facts, the paper's patch
counts and brute force."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from rdr_inputs import make_config, freudenthal, boundary_mask, HGRAD, HCURL
from oracle.solver import Oracle
from oracle.mesh import Topology
from oracle.refelem import element, reference_matrices, tabulate
from oracle.simplex import reference_tet, TET_EDGES
from oracle.fem import tet_quadrature
from oracle.xprec import LD


def _oracle(n, p, space, bc="all", perturb=False, seed=0, coeffs="one", assemble=True):
    c = make_config(0, n=n, p=p, space=space, bc=bc, perturb=perturb, coeffs=coeffs, seed=seed)
    return c, Oracle(c.vertices, c.tets, p, space, c.alpha, c.beta, c.mask, assemble=assemble)


# ------------------------------------------------------------------ mesh
@pytest.mark.parametrize("n", [1, 2, 3])
def test_freudenthal_counts(n):
    """V=(n+1)^3, E=7n^3+9n^2+3n, F=12n^3+6n^2, T=6n^3, 12n^2 boundary faces;
    interior vertex star = 24 cells, 14 edges, 36 faces."""
    v, t, lat = freudenthal(n)
    topo = Topology(v, t, np.zeros((len(t), 4), np.uint8))
    assert (topo.nv, topo.ne, topo.nf, topo.nt) == ((n + 1) ** 3, 7 * n ** 3 + 9 * n ** 2 + 3 * n,
                                                    12 * n ** 3 + 6 * n ** 2, 6 * n ** 3)
    assert topo.boundary_face.sum() == 12 * n ** 2
    if n >= 2:
        c = 1 + (n + 1) * (1 + (n + 1))  # vertex (1,1,1)
        assert (topo.cells == c).any(axis=1).sum() == 24
        assert (topo.edges == c).any(axis=1).sum() == 14
        assert (topo.faces == c).any(axis=1).sum() == 36
    mask = boundary_mask(t, lat, n, "all")
    assert mask.sum() == 12 * n ** 2


def test_cg_dof_count_on_freudenthal():
    for n, p in ((2, 3), (2, 4), (3, 2)):
        c, o = _oracle(n, p, HGRAD, assemble=False)
        assert o.n_total == (n * p + 1) ** 3


# ------------------------------------------------------------------ element level
@pytest.mark.parametrize("space,p", [("hgrad", 3), ("hgrad", 5), ("hcurl", 2), ("hcurl", 4)])
def test_reference_congruent_cell(space, p):
    """S:337 / Lemma 4.4: on a mesh that IS T-hat (vertex order 0..3), the
    quadrature-assembled A equals beta M-hat + alpha K-hat from exact integration."""
    T = reference_tet()
    v = T.coords.astype(float)
    tets = np.array([[0, 1, 2, 3]], dtype=np.int32)
    alpha, beta = np.array([1.7]), np.array([0.3])
    o = Oracle(v, tets, p, space, alpha, beta, np.zeros((1, 4), np.uint8))
    el = element(space, p)
    M, K = reference_matrices(el)
    if space == "hgrad":
        Aref = 0.3 * M.astype(float) + 1.7 * sum(K[a, a] for a in range(3)).astype(float)
    else:
        Aref = 0.3 * sum(M[a, a] for a in range(3)).astype(float) + 1.7 * sum(K[a, a] for a in range(3)).astype(float)
    dm = o.num.dofmap[0]
    A = o.A.toarray()[np.ix_(dm, dm)]
    assert np.abs(A - Aref).max() < 1e-12 * np.abs(Aref).max()
    if space == "hgrad" and p >= 4:
        I = el.interior
        assert np.allclose(np.diag(A)[I], 1.7 + 0.3 * el.lam_cell.astype(float), rtol=1e-12)


def test_p1_textbook_elements():
    """p=1: P1 stiffness |T| grad l_i . grad l_j, mass |T|(1+d_ij)/20; Whitney
    curl-curl |T| 4 (gl_a x gl_b).(gl_c x gl_d) and Whitney mass (textbook)."""
    rng = np.random.default_rng(3)
    v = np.eye(4, 3) * 0 + rng.standard_normal((4, 3))
    tets = np.array([[0, 1, 2, 3]], dtype=np.int32)
    E = (v[1:] - v[0]).T
    vol = abs(np.linalg.det(E)) / 6
    gl = np.zeros((4, 3))
    gl[1:] = np.linalg.inv(E)
    gl[0] = -gl[1:].sum(axis=0)
    Mlam = vol * (np.ones((4, 4)) + np.eye(4)) / 20
    o = Oracle(v, tets, 1, "hgrad", np.array([2.0]), np.array([0.5]), np.zeros((1, 4), np.uint8))
    ref = 0.5 * Mlam + 2.0 * vol * gl @ gl.T
    assert np.abs(o.A.toarray() - ref).max() < 1e-13 * np.abs(ref).max()
    o = Oracle(v, tets, 1, "hcurl", np.array([2.0]), np.array([0.5]), np.zeros((1, 4), np.uint8))
    ref = np.zeros((6, 6))
    for i, (a, b) in enumerate(TET_EDGES):
        for j, (c, d) in enumerate(TET_EDGES):
            m = (Mlam[a, c] * gl[b] @ gl[d] - Mlam[a, d] * gl[b] @ gl[c]
                 - Mlam[b, c] * gl[a] @ gl[d] + Mlam[b, d] * gl[a] @ gl[c])
            k = vol * 4 * np.cross(gl[a], gl[b]) @ np.cross(gl[c], gl[d])
            ref[i, j] = 0.5 * m + 2.0 * k
    assert np.abs(o.A.toarray() - ref).max() < 1e-13 * np.abs(ref).max()


# ------------------------------------------------------------------ global identities
@pytest.mark.parametrize("p", [2, 3, 5])
def test_hgrad_constants_and_volume(p):
    """No Gamma_D: K 1_V = 0 (Lemma 4.1: the constant is 1 on vertex dofs, 0 on
    bubbles); 1_V^T M 1_V = |Omega| = 1 (boundary vertices fixed by the perturbation)."""
    c = make_config(0, n=2, p=p, space=HGRAD, bc="none", perturb=True)
    nt = len(c.tets)
    oK = Oracle(c.vertices, c.tets, p, HGRAD, np.ones(nt), np.zeros(nt), c.mask)
    oM = Oracle(c.vertices, c.tets, p, HGRAD, np.zeros(nt), np.ones(nt), c.mask)
    one = np.zeros(oK.n_total)
    one[:oK.topo.nv] = 1
    assert np.abs(oK.A @ one).max() < 1e-12 * abs(oK.A).max()
    assert abs(one @ (oM.A @ one) - 1.0) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_hcurl_gradients(p):
    """No Gamma_D: K1 G = 0 (curl grad = 0, Lemma 4.3 / Eq. 4.8); G^T M1 G = K0 (the
    H(grad) stiffness); (G xbar)^T M1 (G xbar) = |Omega| with xbar = vertex x-coords."""
    c = make_config(0, n=2, p=p, space=HCURL, bc="none", perturb=True)
    nt = len(c.tets)
    oK = Oracle(c.vertices, c.tets, p, HCURL, np.ones(nt), np.zeros(nt), c.mask)
    oM = Oracle(c.vertices, c.tets, p, HCURL, np.zeros(nt), np.ones(nt), c.mask)
    G = oK._build_gradient()
    K1G = (oK.A @ G)
    assert abs(K1G).max() < 1e-11 * abs(oK.A).max()
    o0 = Oracle(c.vertices, c.tets, p, HGRAD, np.ones(nt), np.zeros(nt), c.mask)
    GMG = (G.T @ oM.A @ G).toarray()
    assert np.abs(GMG - o0.A.toarray()).max() < 1e-11 * abs(o0.A).max()
    xbar = np.zeros(G.shape[1])
    xbar[:oK.topo.nv] = c.vertices[:, 0]
    u = G @ xbar
    assert abs(u @ (oM.A @ u) - 1.0) < 1e-12


def _lagrange_operator(vertices, cells, p, alpha, beta):
    """Independent P_p assembly in a NODAL basis: per cell, monomials in x,y,z of
    degree <= p, Vandermonde at the cell's lattice nodes, physical quadrature."""
    from itertools import product
    exps = [e for e in product(range(p + 1), repeat=3) if sum(e) <= p]
    lam, w = tet_quadrature(2 * p)
    lat = [a for a in product(range(p + 1), repeat=4) if sum(a) == p]
    nodes = {}
    rows, cols, vals = [], [], []
    for ci, cell in enumerate(cells):
        x = vertices[cell]
        pts = np.array([np.array(a) @ x / p for a in lat])
        ids = []
        for pt in pts:
            key = tuple(np.round(pt * 1e9).astype(np.int64))
            ids.append(nodes.setdefault(key, len(nodes)))
        V = np.array([[np.prod(pt ** np.array(e)) for e in exps] for pt in pts])
        Ci = np.linalg.inv(V)          # columns: nodal basis in monomial coefficients
        qp = lam @ x
        vol = abs(np.linalg.det((x[1:] - x[0]).T)) / 6
        Mo = np.array([[np.prod(q ** np.array(e)) for e in exps] for q in qp])
        Gm = np.zeros((len(qp), len(exps), 3))
        for k, e in enumerate(exps):
            for d in range(3):
                if e[d] > 0:
                    ee = list(e)
                    ee[d] -= 1
                    Gm[:, k, d] = e[d] * np.prod(qp ** np.array(ee), axis=1)
        phi = Mo @ Ci
        gphi = np.einsum("qkd,kn->qnd", Gm, Ci)
        Ae = vol * (beta[ci] * np.einsum("q,qi,qj->ij", w, phi, phi)
                    + alpha[ci] * np.einsum("q,qid,qjd->ij", w, gphi, gphi))
        for a in range(len(ids)):
            for b in range(len(ids)):
                rows.append(ids[a]); cols.append(ids[b]); vals.append(Ae[a, b])
    import scipy.sparse as sp
    N = len(nodes)
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N)).toarray(), nodes


@pytest.mark.parametrize("p", [2, 3])
def test_span_change_of_basis(p):
    """north_star pin: the new basis spans P_p conformingly: A_new = T^T A_lagr T with
    T[node, j] = phi_j(node) (6-tet cube, no Dirichlet, random alpha, beta)."""
    c = make_config(0, n=1, p=p, space=HGRAD, bc="none", coeffs="loguniform")
    o = Oracle(c.vertices, c.tets, p, HGRAD, c.alpha, c.beta, c.mask)
    cells = o.topo.cells
    AL, nodes = _lagrange_operator(c.vertices, cells, p, c.alpha, c.beta)
    el = element("hgrad", p)
    Tm = np.zeros((len(nodes), o.n_total))
    for ci, cell in enumerate(cells):
        x = c.vertices[cell]
        from itertools import product
        lat = [a for a in product(range(p + 1), repeat=4) if sum(a) == p]
        bary = np.array(lat, dtype=float) / p
        val = tabulate(el, bary.astype(LD))[0].astype(float)
        for k, a in enumerate(lat):
            pt = np.array(a) @ x / p
            nid = nodes[tuple(np.round(pt * 1e9).astype(np.int64))]
            Tm[nid, o.num.dofmap[ci]] = val[k]
    assert np.linalg.matrix_rank(Tm) == o.n_total
    Anew = o.A.toarray()
    assert np.abs(Tm.T @ AL @ Tm - Anew).max() < 1e-11 * np.abs(Anew).max()


@pytest.mark.parametrize("p", [2, 3])
def test_ned_tangential_conformity(p):
    """Global Ned1 functions have continuous tangential traces across interior faces."""
    c = make_config(0, n=1, p=p, space=HCURL, bc="none", perturb=False)
    o = Oracle(c.vertices, c.tets, p, HCURL, c.alpha, c.beta, c.mask, assemble=False)
    el = element("hcurl", p)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(o.n_total)
    t = o.topo
    face_cells = {}
    for ci in range(t.nt):
        for lf in range(4):
            face_cells.setdefault(t.cell_faces[ci, lf], []).append((ci, lf))
    from oracle.simplex import TET_FACES
    Jh = o.asm
    n_checked = 0
    for f, lst in face_cells.items():
        if len(lst) != 2:
            continue
        pts = rng.dirichlet(np.ones(3), 5)
        vals = []
        for ci, lf in lst:
            bary = np.zeros((5, 4))
            bary[:, list(TET_FACES[lf])] = pts
            phi = tabulate(el, bary.astype(LD))[0].astype(float)
            J = Jh.jacobians(np.array([ci]))[0]
            phys = np.einsum("ab,qnb->qna", np.linalg.inv(J.T), phi)
            vals.append(np.einsum("qna,n->qa", phys, u[o.num.dofmap[ci]]))
        xf = c.vertices[t.faces[f]]
        nrm = np.cross(xf[1] - xf[0], xf[2] - xf[0])
        nrm /= np.linalg.norm(nrm)
        d = vals[0] - vals[1]
        tang = d - (d @ nrm)[:, None] * nrm[None]
        assert np.abs(tang).max() < 1e-10 * np.abs(vals[0]).max()
        n_checked += 1
    assert n_checked == 6  # 18 faces, 12 on the boundary


# ------------------------------------------------------------------ preconditioner / PCG
def test_patch_sizes_table1():
    """P:1783-1787 and Table 1: interior vertex-star interface patch 151 (p=4),
    1423 (p=10); H(curl) recommended split: vertex 151/1423, edge 55/325."""
    for p, vdim, edim in ((4, 151, 55), (10, 1423, 325)):
        c, o = _oracle(3, p, HGRAD, bc="none", assemble=False)
        assert max(len(i) for k, i in o.patch_sets()) == vdim
        c, o = _oracle(3, p, HCURL, bc="none", assemble=False)
        ps = o.patch_sets()
        assert max(len(i) for k, i in ps if k == "pot") == vdim
        assert max(len(i) for k, i in ps if k == "dof") == edim
        # interior edge-star formula 1 + m(p-1)(p+2)/2, m = 6 or 4
        sizes = {len(i) for k, i in ps if k == "dof"}
        assert 1 + 4 * (p - 1) * (p + 2) // 2 in sizes


def test_config_patch_counts():
    """config 1 has 27 patches (max 65); config 2 729 (max 431)."""
    c = make_config(1)
    o = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, assemble=False)
    ps = o.patch_sets()
    assert len(ps) == 27 and max(len(i) for _, i in ps) == 65
    c = make_config(2)
    o = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, assemble=False)
    ps = o.patch_sets()
    assert len(ps) == 729 and max(len(i) for _, i in ps) == 431


@pytest.mark.parametrize("space,n,p", [(HGRAD, 2, 3), (HCURL, 2, 2), (HCURL, 2, 3)])
def test_preconditioner_symmetric_positive(space, n, p):
    c, o = _oracle(n, p, space, perturb=True)
    rng = np.random.default_rng(1)
    x, y = o.mask(rng.standard_normal(o.n_total)), o.mask(rng.standard_normal(o.n_total))
    px, py = o.precond(x), o.precond(y)
    assert abs(x @ py - y @ px) < 1e-13 * np.linalg.norm(x) * np.linalg.norm(px)
    assert x @ px > 0
    # with all-ones weights the additive operator dominates A^-1: x^T P^-1 x >= ... just positivity per sample
    for _ in range(5):
        v = o.mask(rng.standard_normal(o.n_total))
        assert v @ o.precond(v) > 0


def test_single_patch_exact():
    """n=2, p=1, full Dirichlet: one free vertex = one 1x1 patch, so P^-1 = A^-1 and PCG
    takes 1 iteration."""
    c, o = _oracle(2, 1, HGRAD)
    assert o.free.sum() == 1
    b = o.mask(np.ones(o.n_total))
    x, it, res = o.solve(b)
    assert it == 1 and res < 1e-14


@pytest.mark.parametrize("space,n,p", [(HGRAD, 2, 3), (HCURL, 2, 2), (HCURL, 2, 3)])
def test_pcg_matches_dense_solve(space, n, p):
    """PCG at rtol 1e-8 agrees with numpy.linalg.solve to <= 1e-6 relative."""
    c, o = _oracle(n, p, space, perturb=(space == HCURL))
    b = o.mask(c.draw_vector(o.n_total))
    x, it, res = o.solve(b, rtol=1e-8)
    F = o.free
    xd = np.linalg.solve(o.A.toarray()[np.ix_(F, F)], b[F])
    assert np.linalg.norm(x[F] - xd) / np.linalg.norm(xd) < 1e-6
    assert res < 1e-5


def test_config1_iterations():
    """Oracle authority for config 1 (SURVEY F13 probe: ~15, basis not canonicalized)."""
    c = make_config(1)
    o = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = o.mask(c.draw_vector(o.n_total))
    x, it, res = o.solve(b)
    assert 12 <= it <= 18


@pytest.mark.parametrize("p", [4, 6])
def test_lemma47_weak_couplings(p):
    """Lemma 4.7: per-cell kappa(P_T^-1 A_T), P_T = blockdiag(diag A_II, A_GG),
    is O(1) on a Kuhn tet with h = 1/8 (survey reference 3.3 / 4.2 at p=4 / 6);
    on the reference-congruent cell with beta = 0, A_T - P_T = 0 entrywise."""
    import scipy.linalg as sla
    v, t, _ = freudenthal(1)
    v = v / 8
    o = Oracle(v, t[:1], p, HGRAD, np.ones(1), np.ones(1), np.zeros((1, 4), np.uint8))
    dm = o.num.dofmap[0]
    A = o.A.toarray()[np.ix_(dm, dm)]
    I = element("hgrad", p).interior
    P = A.copy()
    P[np.ix_(I, ~I)] = 0
    P[np.ix_(~I, I)] = 0
    AI = P[np.ix_(I, I)]
    P[np.ix_(I, I)] = np.diag(np.diag(AI))
    ev = sla.eigvalsh(A, P)
    kappa = ev[-1] / ev[0]
    assert 1.0 < kappa < 10.0
    T = reference_tet()
    o = Oracle(T.coords.astype(float), np.array([[0, 1, 2, 3]]), p, HGRAD, np.ones(1), np.zeros(1),
               np.zeros((1, 4), np.uint8))
    A = o.A.toarray()[np.ix_(o.num.dofmap[0], o.num.dofmap[0])]
    P = A.copy()
    P[np.ix_(I, ~I)] = 0
    P[np.ix_(~I, I)] = 0
    P[np.ix_(I, I)] = np.diag(np.diag(A[np.ix_(I, I)]))
    assert np.abs(A - P).max() < 1e-12 * np.abs(A).max()


# ------------------------------------------------------------------ manufactured solutions
def _mms_errors(space, n, p):
    c = make_config(0, n=n, p=p, space=space, bc="all")
    o = Oracle(c.vertices, c.tets, p, space, c.alpha, c.beta, c.mask)
    asm = o.asm
    pi = math.pi
    lam, w = tet_quadrature(2 * p + 4)
    el = element(o.space, p)
    val, der = [x.astype(float) for x in tabulate(el, lam.astype(LD))]
    cells = np.arange(o.topo.nt)
    J = asm.jacobians(cells)
    det = np.linalg.det(J)
    x0 = c.vertices[o.topo.cells[:, 0]]
    Vh = asm.Vhat
    xq = x0[:, None, :] + np.einsum("cab,qb->cqa", J, lam @ Vh - Vh[0])
    X, Y, Z = xq[..., 0], xq[..., 1], xq[..., 2]
    vol = np.abs(det) * asm.vol_hat
    s = np.sin
    if space == HGRAD:
        u = s(pi * X) * s(pi * Y) * s(pi * Z)
        f = (1 + 3 * pi ** 2) * u
        Fe = np.einsum("c,q,cq,qn->cn", vol, w, f, val)
    else:
        u = np.stack([s(pi * Y) * s(pi * Z), s(pi * X) * s(pi * Z), s(pi * X) * s(pi * Y)], axis=-1)
        # curl curl u = 2 pi^2 u for this field
        f = (1 + 2 * pi ** 2) * u
        Jit = np.linalg.inv(np.transpose(J, (0, 2, 1)))
        ph = np.einsum("cab,qnb->cqna", Jit, val)
        Fe = np.einsum("c,q,cqa,cqna->cn", vol, w, f, ph)
    b = np.zeros(o.n_total)
    np.add.at(b, o.num.dofmap, Fe)
    b = o.mask(b)
    F = o.free
    x = np.zeros(o.n_total)
    x[F] = spla.spsolve(o.A[F][:, F].tocsc(), b[F])
    xe = x[o.num.dofmap]
    if space == HGRAD:
        uh = np.einsum("qn,cn->cq", val, xe)
        return math.sqrt(np.einsum("c,q,cq->", vol, w, (uh - u) ** 2))
    uh = np.einsum("cqna,cn->cqa", ph, xe)
    return math.sqrt(np.einsum("c,q,cqa->", vol, w, (uh - u) ** 2))


@pytest.mark.parametrize("space,p,rate,n", [(HGRAD, 1, 2, 4), (HGRAD, 2, 3, 2), (HGRAD, 3, 4, 2),
                                            (HCURL, 1, 1, 4), (HCURL, 2, 2, 2), (HCURL, 3, 3, 2)])
def test_mms_convergence(space, p, rate, n):
    """Textbook a-priori rates: CG_p L2 ~ h^{p+1}; Ned1_p L2 ~ h^p (meshes n -> 2n)."""
    e1 = _mms_errors(space, n, p)
    e2 = _mms_errors(space, 2 * n, p)
    assert math.log2(e1 / e2) >= rate - 0.2


def test_unsplit_preconditioner_exactness_and_pcg():
    """Unsplit one-level decompositions: symmetric, positive,
    and PCG agrees with a dense solve (both spaces)."""
    import scipy.sparse.linalg  # noqa: F401
    for space, p in ((HGRAD, 3), (HCURL, 2)):
        c = make_config(0, n=2, p=p, space=space, perturb=True, bc="x0", coeffs="loguniform")
        o = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition="unsplit")
        rng = np.random.default_rng(3)
        x, y = o.mask(rng.standard_normal(o.n_total)), o.mask(rng.standard_normal(o.n_total))
        px, py = o.precond(x), o.precond(y)
        assert abs(x @ py - y @ px) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(py)
        assert x @ px > 0
        b = o.mask(c.draw_vector(o.n_total))
        xs, it, res = o.solve(b, rtol=1e-10)
        A = o.A.toarray()[np.ix_(o.free, o.free)]
        xd = np.linalg.solve(A, b[o.free])
        assert np.linalg.norm(xs[o.free] - xd) <= 1e-7 * np.linalg.norm(xd)
