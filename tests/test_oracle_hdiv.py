"""Pins of the H(div) oracle: the RT_p reference element of
Eq. 3.17-3.18 and the PAFW1(X2_Gamma) + J(X2_I) preconditioner
(Eq. 5.16), against what the paper and the mathematics fix:

* dimensions p(p+1)(p+3)/2 and the per-entity counts of Eq. 3.18;
* Lemma 4.1: the face-Whitney basis functions ARE the Whitney
  2-forms 2(l_i dl_j^dl_k - l_j dl_i^dl_k + l_k dl_i^dl_j);
* Lemma 4.3: curl of every type-I Ned1_p face / cell basis
  function is the RT_p type-II basis function with the same index, and curl of
  a Ned1_p Whitney edge function is the signed sum of the face-Whitney
  functions of the faces containing the edge (exact sequence, Eq. 2.4);
* Lemma 4.4: the interior blocks of K-hat = I / 0 and of
  M-hat = diag(lambda) / I, zero interior-interface coupling of K-hat;
* the divergence theorem: int div phi_j = +-1 for the face-Whitney functions
  (sign = orientation of the sorted face vs the outward normal), 0 otherwise;
* physical-quadrature assembly on an affine cell equals the exact contraction
  of the reference matrices with the Piola factors J^T J / |det J|, 1/|det J|;
* normal (not tangential) continuity of global RT_p fields across interior
  faces of a perturbed mesh; Eq. 3.17 re-checked by quadrature;
* globally, with the discrete curl C (face/edge incidence + type-I -> type-II):
  K2 C = 0 and C^T M2 C = the Ned1 curl-curl operator;
* the global operator is SPD, PCG converges, sampled rows equal global rows,
  and the hybrid Schwarz with the exact W^2 coarse solve needs 1 iteration at
  p = 1 (RT_1 = W^2).
"""
import numpy as np
import pytest

from rdr_inputs import make_config
from oracle.refelem import rt_element, ned_element, reference_matrices, tabulate, rt_bubbles
from oracle.simplex import reference_tet, TET_FACES, TET_EDGES

PTS = np.random.default_rng(11).dirichlet(np.ones(4), 9).astype(np.longdouble)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_rt_dimensions(p):
    el = rt_element(p)
    assert el.n == p * (p + 1) * (p + 3) // 2
    ents = el.dof_entity
    per_face = sum(1 for e in ents if e[0] == 2 and e[1] == 0)
    assert per_face == p * (p + 1) // 2                       # dim P_{p-1}(F)
    assert sum(1 for e in ents if e[0] == 3) == (p + 1) * p * (p - 1) // 2
    assert sum(1 for e in ents if e[0] == 3 and e[3] == "I") == p * (p + 1) * (p + 2) // 6 - 1  # div onto P_{p-1}/R
    assert len(rt_bubbles(p).lam) == p * (p + 1) * (p + 2) // 6 - 1
    assert np.all(np.diff(rt_bubbles(p).lam.astype(float)) <= 0)  # R-A5: descending lambda


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_rt_face_whitney_functions(p):
    el = rt_element(p)
    T = reference_tet()
    val, _ = tabulate(el, PTS)
    g = T.g.astype(np.float64)
    lam = PTS.astype(np.float64)
    for f, (i, j, k) in enumerate(TET_FACES):
        w = 2 * (lam[:, [i]] * np.cross(g[j], g[k]) - lam[:, [j]] * np.cross(g[i], g[k])
                 + lam[:, [k]] * np.cross(g[i], g[j]))
        col = el.dof_entity.index((2, f, 0, "W"))
        assert np.abs(val[:, col].astype(np.float64) - w).max() <= 1e-13


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_rt_d_preserves_basis_functions(p):
    rt, ned = rt_element(p), ned_element(p)
    val, _ = tabulate(rt, PTS)
    _, curl = tabulate(ned, PTS)
    val, curl = val.astype(np.float64), curl.astype(np.float64)
    for a, (dim, e, j, typ) in enumerate(ned.dof_entity):
        if dim >= 2 and typ == "I":          # Lemma 4.3: curl phi^{1,I}_{S,j} = phi^{2,II}_{S,j}
            b = rt.dof_entity.index((dim, e, j, "II"))
            assert np.abs(curl[:, a] - val[:, b]).max() <= 1e-12
        elif dim == 1 and typ == "W":        # curl w_E = sum_{F > E} [F:E] w_F
            ea, eb = TET_EDGES[e]
            expect = np.zeros_like(curl[:, a])
            for f, tri in enumerate(TET_FACES):
                if ea in tri and eb in tri:
                    c = [x for x in tri if x not in (ea, eb)][0]
                    # boundary of the oriented face (t0,t1,t2): +[t1t2] - [t0t2] + [t0t1]
                    pos = tri.index(c)
                    sign = (-1) ** pos
                    expect += sign * val[:, rt.dof_entity.index((2, f, 0, "W"))]
            assert np.abs(curl[:, a] - expect).max() <= 1e-12
        elif typ == "II":                    # curl grad = 0
            assert np.abs(curl[:, a]).max() <= 1e-11


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_rt_reference_matrix_structure(p):
    el = rt_element(p)
    M, K = reference_matrices(el)
    M, K = M.astype(np.float64), K.astype(np.float64)
    Mt = M[0, 0] + M[1, 1] + M[2, 2]
    ents = el.dof_entity
    interior = np.array([e[0] == 3 for e in ents])
    tI = np.array([e[3] == "I" for e in ents])
    tII = np.array([e[3] == "II" for e in ents])
    iI, iII, gam = np.nonzero(interior & tI)[0], np.nonzero(interior & tII)[0], np.nonzero(~interior)[0]
    s = np.abs(K).max()
    assert np.abs(K[np.ix_(iI, iI)] - np.eye(len(iI))).max(initial=0) <= 1e-13 * max(1, s)
    assert np.abs(K[tII]).max(initial=0) <= 1e-13 * s
    assert np.abs(K[np.ix_(np.nonzero(interior)[0], gam)]).max(initial=0) <= 1e-13 * s
    assert np.abs(Mt[np.ix_(iI, iI)] - np.diag(el.lam_cell.astype(np.float64))).max(initial=0) <= 1e-14
    assert np.abs(Mt[np.ix_(iII, iII)] - np.eye(len(iII))).max(initial=0) <= 1e-13
    assert np.abs(Mt[np.ix_(iII, gam)]).max(initial=0) <= 1e-13
    assert np.allclose(M, np.transpose(M, (1, 0, 3, 2)), atol=1e-14)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_rt_divergence_theorem(p):
    el = rt_element(p)
    T = reference_tet()
    # int_T div phi_j by exact integration of the divergence polynomial
    Dv = (el.C.T @ (el.span @ T.div_op(p)))
    ones = np.ones((1, 1), dtype=np.longdouble)
    intdiv = (Dv @ T.I(p - 1, 0) @ ones.T)[:, 0].astype(np.float64)
    x = T.coords.astype(np.float64)
    for j, (dim, e, jj, typ) in enumerate(el.dof_entity):
        expect = 0.0
        if dim == 2 and typ == "W":
            i0, i1, i2 = TET_FACES[e]
            opp = [v for v in range(4) if v not in (i0, i1, i2)][0]
            n_sorted = np.cross(x[i1] - x[i0], x[i2] - x[i0])
            expect = 1.0 if n_sorted @ (x[i0] - x[opp]) > 0 else -1.0
        assert abs(intdiv[j] - expect) <= 1e-13


def test_rt_physical_assembly_matches_piola_contraction():
    from oracle.mesh import Topology, number, dof_layout
    from oracle.fem import Assembler
    p = 3
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 3))
    topo = Topology(x, np.array([[2, 0, 3, 1]]), np.zeros((1, 4), dtype=np.uint8))
    num = number("hdiv", p, topo, dof_layout("hdiv", p))
    asm = Assembler("hdiv", p, topo, num)
    alpha, beta = np.array([0.7]), np.array([1.9])
    Ae = asm.element_matrices(np.array([0]), alpha, beta)[0]
    J = asm.jacobians(np.array([0]))[0]
    ad = abs(np.linalg.det(J))
    M, K = reference_matrices(rt_element(p))
    G = J.T @ J
    ref = sum(beta[0] * G[a, b] / ad * M[a, b].astype(np.float64) for a in range(3) for b in range(3))
    ref = ref + alpha[0] / ad * K.astype(np.float64)
    assert np.abs(Ae - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_hdiv_global_operator_and_pcg(p):
    from oracle.solver import Oracle
    from oracle.sampled import SampledOracle
    c = make_config(0, n=2, p=p, space=1, perturb=True, bc="x0", coeffs="loguniform")
    O = Oracle(c.vertices, c.tets, p, "hdiv", c.alpha, c.beta, c.mask)
    A = O.A.toarray()
    f = O.free
    assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    assert np.linalg.eigvalsh(A[np.ix_(f, f)])[0] > 0
    # Dirichlet (R-A11 for 2-forms): exactly the dofs of Gamma_D faces are constrained
    assert np.array_equal(~f, np.isin(O.num.entity[:, 1], np.nonzero(O.topo.dir_face)[0]) & (O.num.entity[:, 0] == 2))
    b = c.draw_vector(O.n_total)
    x, it, res = O.solve(b, rtol=1e-10)
    assert res <= 1e-6 and it < 200
    S = SampledOracle(c.vertices, c.tets, p, "hdiv", c.alpha, c.beta, c.mask)
    rows = np.arange(0, O.n_total, 5)
    r = c.draw_vector(O.n_total)
    y = O.apply(r)
    assert np.abs(S.apply_rows(r, rows) - y[rows]).max() <= 1e-12 * np.abs(y).max()
    z = O.precond(r)
    assert np.abs(S.precond_rows(r, rows) - z[rows]).max() <= 1e-12 * np.abs(z).max()


def test_hdiv_hybrid_exact_at_p1():
    """RT_1 = W^2: the hybrid sweep's exact coarse solve is the whole space."""
    from oracle.hybrid import HybridOracle
    c = make_config(0, n=2, p=1, space=1, perturb=True, bc="x0", coeffs="loguniform")
    H = HybridOracle(c.vertices, c.tets, 1, "hdiv", c.alpha, c.beta, c.mask)
    _, it, res = H.solve(c.draw_vector(H.n_total))
    assert it == 1 and res <= 1e-12


@pytest.mark.parametrize("p", [1, 2, 3])
def test_rt_normal_conformity(p):
    """Global RT_p functions (Piola phi = J phi-hat / det J, sorted-vertex face
    orientation, DESIGN.md R-D2) have continuous normal traces across interior
    faces of a perturbed mesh, for a random coefficient vector; the tangential
    traces do jump (so the check is not vacuous)."""
    from oracle.solver import Oracle
    from oracle.xprec import LD
    c = make_config(0, n=2, p=p, space=2, bc="none", perturb=True)
    o = Oracle(c.vertices, c.tets, p, "hdiv", c.alpha, c.beta, c.mask, assemble=False)
    el = rt_element(p)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(o.n_total)
    t = o.topo
    face_cells = {}
    for ci in range(t.nt):
        for lf in range(4):
            face_cells.setdefault(t.cell_faces[ci, lf], []).append((ci, lf))
    n_checked, tang_jump = 0, 0.0
    for f, lst in face_cells.items():
        if len(lst) != 2:
            continue
        pts = rng.dirichlet(np.ones(3), 4)
        vals = []
        for ci, lf in lst:
            bary = np.zeros((4, 4))
            bary[:, list(TET_FACES[lf])] = pts
            phi = tabulate(el, bary.astype(LD))[0].astype(float)
            J = o.asm.jacobians(np.array([ci]))[0]
            phys = np.einsum("ab,qnb->qna", J, phi) / np.linalg.det(J)
            vals.append(np.einsum("qna,n->qa", phys, u[o.num.dofmap[ci]]))
        xf = c.vertices[t.faces[f]]
        nrm = np.cross(xf[1] - xf[0], xf[2] - xf[0])
        nrm /= np.linalg.norm(nrm)
        d = vals[0] - vals[1]
        assert np.abs(d @ nrm).max() < 1e-10 * np.abs(vals[0]).max()
        tang_jump = max(tang_jump, np.abs(d - (d @ nrm)[:, None] * nrm[None]).max())
        n_checked += 1
    assert n_checked > 0 and tang_jump > 1e-3


@pytest.mark.parametrize("p", [2, 3, 4])
def test_rt_eigen_orthogonality_by_quadrature(p):
    """Eq. 3.17 re-checked by the tet quadrature of oracle/fem.py (exact to degree
    2p+2, independent of the closed-form monomial integrals the construction
    uses): (div Phi_i, div Phi_j) = delta_ij, (Phi_i, Phi_j) = lambda_j delta_ij."""
    from oracle.fem import tet_quadrature
    T = reference_tet()
    E = rt_bubbles(p)
    lam, w = tet_quadrature(2 * p + 2)
    bary = lam.astype(np.longdouble)
    vals = T.eval2(E.F, p, bary).astype(float)                      # [q, n, 3]
    divs = T.eval0(E.F @ T.div_op(p), p - 1, bary).astype(float)    # [q, n]
    vol = float(T.vol)
    M = vol * np.einsum("q,qia,qja->ij", w, vals, vals)
    K = vol * np.einsum("q,qi,qj->ij", w, divs, divs)
    assert np.abs(K - np.eye(len(E.lam))).max() <= 1e-12
    assert np.abs(M - np.diag(E.lam.astype(float))).max() <= 1e-12 * max(1.0, float(E.lam.max()))


def _discrete_curl(o_rt, o_ned, p):
    """C: Ned1_p dofs -> RT_p dofs (Lemma 4.1 + 4.3): C[W(F), W(E)] = [F:E] (the
    sign of E in the boundary of the sorted face (a,b,c): +bc -ac +ab) and
    C[typeII(S,j), typeI(S,j)] = 1 for S = faces, cell."""
    import scipy.sparse as sp
    t, rt, ned = o_rt.topo, o_rt.num, o_ned.num
    rows, cols, vals = [], [], []
    for f, (a, b, cc) in enumerate(t.faces):
        wf = rt.offsets[2] + f * rt.per[2]
        for (x, y), sgn in (((b, cc), 1.0), ((a, cc), -1.0), ((a, b), 1.0)):
            rows.append(wf)
            cols.append(ned.offsets[1] + t.edge_index[(x, y)] * ned.per[1])
            vals.append(sgn)
        nIf = ned.per[2] - (p - 1) * (p - 2) // 2           # Ned1 type-I face dofs = RT type-II face dofs
        for j in range(nIf):
            rows.append(wf + 1 + j)
            cols.append(ned.offsets[2] + f * ned.per[2] + j)
            vals.append(1.0)
    nIc_ned = ned.per[3] - (p - 1) * (p - 2) * (p - 3) // 6   # Ned1 type-I cell dofs
    nI_rt = p * (p + 1) * (p + 2) // 6 - 1                   # RT type-I cell dofs precede type-II
    for cidx in range(t.nt):
        for j in range(nIc_ned):
            rows.append(rt.offsets[3] + cidx * rt.per[3] + nI_rt + j)
            cols.append(ned.offsets[3] + cidx * ned.per[3] + j)
            vals.append(1.0)
    return sp.csr_matrix((vals, (rows, cols)), shape=(rt.n_total, ned.n_total))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_hdiv_curls(p):
    """No Gamma_D, on a perturbed mesh: the div-div part annihilates the
    discrete curl, K2 C = 0 (div curl = 0), and C^T M2 C = the Ned1 curl-curl
    operator (curl phi^1 = C phi^2 exactly, Lemma 4.3 globally)."""
    from oracle.solver import Oracle
    c = make_config(0, n=2, p=p, space=2, bc="none", perturb=True)
    nt = len(c.tets)
    oK = Oracle(c.vertices, c.tets, p, "hdiv", np.ones(nt), np.zeros(nt), c.mask)
    oM = Oracle(c.vertices, c.tets, p, "hdiv", np.zeros(nt), np.ones(nt), c.mask)
    o1 = Oracle(c.vertices, c.tets, p, "hcurl", np.ones(nt), np.zeros(nt), c.mask)
    C = _discrete_curl(oK, o1, p)
    assert abs(oK.A @ C).max() < 1e-11 * abs(oK.A).max()
    CMC = (C.T @ oM.A @ C).toarray()
    assert np.abs(CMC - o1.A.toarray()).max() < 1e-11 * abs(o1.A).max()
