"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs. Bars (BASELINE.json north_star): operator and
preconditioner applies within 1e-11 relative l2, PCG iteration counts within
+-1 at rtol 1e-8."""
import numpy as np
import pytest

from rdr_inputs import make_config, HGRAD, HCURL, HDIV

pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _pair(torch, cfg, dec="split", **kw):
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    c = make_config(cfg, **kw)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask,
                   decomposition=rdr.UNSPLIT if dec == "unsplit" else rdr.SPLIT)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=dec)
    assert S.n_total == O.n_total
    return c, S, O


def _check_apply_precond(torch, c, S, O, nvec=2):
    for _ in range(nvec):
        x = c.draw_vector(O.n_total)            # constrained entries NOT zeroed: must be ignored
        xt = torch.from_numpy(x).cuda()
        y = S.apply(xt).cpu().numpy()
        z = S.precond(xt).cpu().numpy()
        ya, za = O.apply(x), O.precond(x)
        assert rel(y, ya) <= TOL, rel(y, ya)
        assert rel(z, za) <= TOL, rel(z, za)
        assert np.all(y[~O.free] == 0) and np.all(z[~O.free] == 0)


# DESIGN.md R-A16 tie: ||z_k|| is not monotone in k, so when the oracle's
# ||z_k|| / ||z_0|| at the earlier of the two exits equals rtol to within TIE
# (relative), both exits satisfy the stopping rule up to rounding and the counts
# may differ by more than one. (RT_4 with log-uniform coefficients: oracle ratio
# 1.00005e-8 at the GPU's exit k = 94.) The rule prints a line when it fires.
TIE = 1e-4


def _check_iters(S, it, ito, ratio_at, rtol=1e-8):
    """+-1 iterations against the oracle's count ito (north_star), after
    checking that the GPU's own exit satisfies R-A16 (||z_k|| <= rtol ||z_0||).
    ratio_at(k): the oracle's ||z_k|| / ||z_0|| (None if unknown)."""
    st = S.last_stats()
    assert st["iters"] == it and st["converged"] == 1
    assert st["z_last"] <= rtol * st["z0"], st
    if abs(it - ito) <= 1:
        return
    k = min(it, ito)
    r = ratio_at(k)
    print(f"R-A16 tie rule fired: gpu {it} iterations, oracle {ito}; oracle ||z_{k}||/||z_0|| = {r}")
    assert r is not None and abs(r / rtol - 1.0) <= TIE, (it, ito, r)


def _check_pcg(torch, c, S, O):
    b = c.draw_vector(O.n_total)
    x, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
    hist = []
    xo, ito, res = O.solve(b, rtol=1e-8, history=hist)
    _check_iters(S, it, ito, lambda k: hist[k - 1] if 0 < k <= len(hist) else None)
    xg = x.cpu().numpy()
    bm = O.mask(b)
    assert np.linalg.norm(bm - O.apply(xg)) / np.linalg.norm(bm) <= 1e-5
    assert rel(xg, xo) <= 1e-6
    return it, ito


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10])
@pytest.mark.parametrize("perturb", [False, True])
def test_hgrad_small(torch_cuda, p, perturb):
    c, S, O = _pair(torch_cuda, 0, n=2, p=p, space=HGRAD, perturb=perturb, bc="all")
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("perturb", [False, True])
def test_hcurl_small(torch_cuda, p, perturb):
    c, S, O = _pair(torch_cuda, 0, n=2, p=p, space=HCURL, perturb=perturb, bc="all")
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


@pytest.mark.parametrize("p,bc", [(10, "x0")])
def test_hcurl_high_p(torch_cuda, p, bc):
    """Ned1_10 (north_star: H(curl) up to p=10) on the 6-tet cube with partial
    Dirichlet, every row against the global oracle (p = 9, 10 with full
    Dirichlet at full size: test_config78_high_p_sampled); the oracle's x87
    reference element dominates the cost at this degree."""
    c, S, O = _pair(torch_cuda, 0, n=1, p=p, space=HCURL, perturb=False, bc=bc)
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


@pytest.mark.parametrize("space,bc,coeffs", [(HGRAD, "x0", "loguniform"), (HCURL, "x0", "loguniform"),
                                             (HGRAD, "none", "one")])
def test_partial_dirichlet_and_contrast(torch_cuda, space, bc, coeffs):
    c, S, O = _pair(torch_cuda, 0, n=3, p=3, space=space, perturb=True, bc=bc, coeffs=coeffs)
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


def test_config1(torch_cuda):
    c, S, O = _pair(torch_cuda, 1)
    b = c.draw_vector(O.n_total)   # the config's rhs (first draw)
    x, it = S.solve(torch_cuda.from_numpy(b).cuda(), rtol=1e-8)
    xo, ito, _ = O.solve(b)
    assert abs(it - ito) <= 1
    _check_apply_precond(torch_cuda, c, S, O)


def test_config2(torch_cuda):
    """BASELINE configs[1] (the bench workload) at full size."""
    c, S, O = _pair(torch_cuda, 2)
    O.build_preconditioner(kappa=False)
    _check_apply_precond(torch_cuda, c, S, O, nvec=1)
    _check_pcg(torch_cuda, c, S, O)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_config5_sweep_small_p(torch_cuda, p):
    """configs[4] at p <= 4: full oracle (every row, PCG run by the oracle)."""
    c, S, O = _pair(torch_cuda, 5, p=p)
    O.build_preconditioner(kappa=False)
    _check_apply_precond(torch_cuda, c, S, O, nvec=1)
    _check_pcg(torch_cuda, c, S, O)


def test_symmetry_and_gradient_kernel(torch_cuda):
    """x^T A y = y^T A x, x^T P^-1 y = y^T P^-1 x through the library; K1 G = 0:
    A(G u) does not depend on alpha (H(curl), no Dirichlet)."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(0, n=2, p=3, space=HCURL, perturb=True, bc="none")
    S = rdr.Solver(c.vertices, c.tets, 3, HCURL, c.alpha, c.beta, c.mask)
    rng = np.random.default_rng(0)
    x, y = (torch.from_numpy(rng.standard_normal(S.n_total)).cuda() for _ in range(2))
    assert abs(float(x @ S.apply(y) - y @ S.apply(x))) <= 1e-12 * float(x.norm() * S.apply(x).norm())
    assert abs(float(x @ S.precond(y) - y @ S.precond(x))) <= 1e-12 * float(x.norm() * S.precond(x).norm())
    from oracle.solver import Oracle
    O = Oracle(c.vertices, c.tets, 3, HCURL, c.alpha, c.beta, c.mask, assemble=False)
    G = O._build_gradient()
    u = G @ rng.standard_normal(G.shape[1])
    ut = torch.from_numpy(u).cuda()
    S2 = rdr.Solver(c.vertices, c.tets, 3, HCURL, 1e3 * c.alpha, c.beta, c.mask)
    a1, a2 = S.apply(ut).cpu().numpy(), S2.apply(ut).cpu().numpy()
    assert rel(a2, a1) <= 1e-10


def test_error_codes(torch_cuda):
    from paper_2506_17406_b200 import rdr
    c = make_config(0, n=1, p=2, space=HGRAD, bc="all")
    bad = c.mask.copy()
    # a mask bit on an interior face
    from oracle.mesh import Topology
    T = Topology(c.vertices, c.tets, np.zeros_like(c.mask))
    t0 = 0
    for i in range(4):
        f = tuple(sorted(np.delete(c.tets[t0], i)))
        fi = {tuple(x): k for k, x in enumerate(T.faces)}[f]
        if not T.boundary_face[fi]:
            bad[t0, i] = 1
            break
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, 2, HGRAD, c.alpha, c.beta, bad)
    assert e.value.code == -2
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, 2, HGRAD, -c.alpha, c.beta, c.mask)
    assert e.value.code == -1
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, 13, HGRAD, c.alpha, c.beta, c.mask)
    assert e.value.code == -1
    v = c.vertices.copy()
    v[c.tets[0, 1]] = v[c.tets[0, 0]]  # collapse an edge
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(v, c.tets, 2, HGRAD, c.alpha, c.beta, c.mask)
    assert e.value.code == -2
    for space in (HCURL, HDIV):  # beta = 0: gradients / div-free fields in the kernel (rdr.h RDR_EINVAL)
        with pytest.raises(rdr.RdrError) as e:
            rdr.Solver(c.vertices, c.tets, 2, space, c.alpha, 0 * c.beta, np.zeros_like(c.mask))
        assert e.value.code == -1
    rdr.Solver(c.vertices, c.tets, 2, HGRAD, c.alpha, 0 * c.beta, c.mask)  # beta = 0 is valid for H(grad)


def test_degenerate_sizes(torch_cuda):
    """n=1 full Dirichlet at p=1: no free dof -> y = 0, z = 0, PCG 0 iterations;
    p=12 H(grad) on one cube (largest supported element)."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(0, n=1, p=1, space=HGRAD, bc="all")
    S = rdr.Solver(c.vertices, c.tets, 1, HGRAD, c.alpha, c.beta, c.mask)
    b = torch.ones(S.n_total, dtype=torch.float64, device="cuda")
    assert float(S.apply(b).abs().max()) == 0.0 and float(S.precond(b).abs().max()) == 0.0
    x, it = S.solve(b)
    assert it == 0 and float(x.abs().max()) == 0.0
    c = make_config(0, n=1, p=12, space=HGRAD, bc="none")
    S = rdr.Solver(c.vertices, c.tets, 12, HGRAD, c.alpha, c.beta, c.mask)
    assert S.info["n_loc"] == 455


# ---------------------------------------------------------------- full-size configs (sampled rows)
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_pcg_iters.json")


def _golden(cfg, p):
    for e in json.load(open(GOLDEN))["entries"]:
        if e["cfg"] == cfg and e["p"] == p:
            return e
    raise KeyError(f"no oracle iteration count for cfg{cfg} p={p} in {GOLDEN} (scripts/oracle_golden.py)")


def _golden_iters(cfg, p):
    return _golden(cfg, p)["iters"]


def _sample_rows(O, n_vertices=3, n_cells=4, seed=1):
    """Rows spanning every dof kind: the star dofs of a few interior vertices
    (vertex, edge, face dofs), the interior dofs of a few cells, constrained dofs."""
    rng = np.random.default_rng(seed)
    t = O.topo
    if O.space == "hdiv":  # edge stars: the face dofs of a few interior edges, cell interiors, constrained
        rows = []
        interior_e = np.nonzero(~t.dir_edge)[0]
        for e in rng.choice(interior_e, min(n_vertices, len(interior_e)), replace=False):
            _, idx = O.edge_patch(int(e))
            rows.extend(rng.choice(idx, min(12, len(idx)), replace=False))
        for c in rng.choice(t.nt, n_cells, replace=False):
            rows.extend(rng.choice(O.num.dofmap[c], 3, replace=False))
        rows.extend(rng.choice(np.nonzero(O.num.constrained)[0], 3, replace=False) if O.num.constrained.any() else [])
        return np.unique(np.asarray(rows, dtype=np.int64))
    interior_v = np.nonzero(~t.dir_vertex)[0]
    verts = rng.choice(interior_v, min(n_vertices, len(interior_v)), replace=False) if len(interior_v) else []
    rows = []
    for v in verts:
        kind, idx = O.vertex_patch(int(v))
        if kind == "pot":  # H(curl): Ned1 dofs of the edges / faces of the star
            idx = np.nonzero(np.abs(O.G[:, idx]).sum(axis=1).A1)[0]
        rows.extend(rng.choice(idx, min(12, len(idx)), replace=False))
    for c in rng.choice(t.nt, n_cells, replace=False):
        rows.extend(rng.choice(O.num.dofmap[c], 3, replace=False))
    rows.extend(rng.choice(np.nonzero(O.num.constrained)[0], 3, replace=False) if O.num.constrained.any() else [])
    return np.unique(np.asarray(rows, dtype=np.int64))


def _check_sampled(torch, c, S, O, rows):
    x = c.draw_vector(O.n_total)
    xt = torch.from_numpy(x).cuda()
    y = S.apply(xt).cpu().numpy()
    z = S.precond(xt).cpu().numpy()
    ya, za = O.apply_rows(x, rows), O.precond_rows(x, rows)
    assert rel(y[rows], ya) <= TOL, rel(y[rows], ya)
    assert rel(z[rows], za) <= TOL, rel(z[rows], za)
    assert np.all(y[~O.free] == 0) and np.all(z[~O.free] == 0)


def _check_sampled_pcg(torch, c, S, O, rows, b, iters_expected=None):
    """PCG on the config's rhs b (its first draw, as in the golden file): converges,
    iterations within +-1 of the oracle's (golden) count, and the stopping rule
    of R-A16 holds on sampled rows with the oracle's own residual and
    preconditioner: ||P^-1 (b - A x)|| <= 1e-6 ||P^-1 b|| there (the global
    criterion is 1e-8 in l2; a row sample gets two decades of slack)."""
    x, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
    assert S.converged
    if iters_expected is not None:
        g = iters_expected if isinstance(iters_expected, dict) else {"iters": iters_expected}
        tail = g.get("z_ratio_tail", [])  # the oracle's last ratios, ending at k = g["iters"]
        _check_iters(S, it, g["iters"], lambda k: tail[len(tail) - 1 - (g["iters"] - k)]
                     if 0 <= g["iters"] - k < len(tail) else None)
    xg = x.cpu().numpy()
    z = O.precond_residual_rows(b, xg, rows)
    z0 = O.precond_rows(b, rows)
    assert np.linalg.norm(z) <= 1e-6 * np.linalg.norm(z0), (np.linalg.norm(z), np.linalg.norm(z0))
    return it


def _sampled_pair(cfg, **kw):
    from paper_2506_17406_b200 import rdr
    from oracle.sampled import SampledOracle
    c = make_config(cfg, **kw)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    O = SampledOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    assert S.n_total == O.n_total
    return c, S, O


def test_config3_sampled(torch_cuda):
    """BASELINE configs[2]: H(grad) p=10 on 16^3 x 6 (4.17 M dofs, 29 GB of patch
    inverses). Oracle rows computed one by one (SURVEY §8(c) config-3 scope)."""
    c, S, O = _sampled_pair(3)
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O)
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b, _golden(3, 10))


def test_config4_sampled(torch_cuda):
    """BASELINE configs[3]: H(curl) Ned1_6 on 12^3 x 6 with the type-I
    potential + edge star patches; PCG iterations vs the oracle's (golden)."""
    c, S, O = _sampled_pair(4)
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O)
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b, _golden(4, 6))


@pytest.mark.parametrize("p", [5, 6, 7, 8, 9, 10, 11, 12])
def test_config5_sweep(torch_cuda, p):
    """BASELINE configs[4]: the p-sweep on the perturbed 8^3 x 6 mesh."""
    c, S, O = _sampled_pair(5, p=p)
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O, n_vertices=2, n_cells=3)
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b, _golden(5, p))


# ---------------------------------------------------------------- ABI semantics on the device
@pytest.mark.parametrize("space", [HGRAD, HCURL, HDIV])
def test_loop_modes_and_profile(torch_cuda, space):
    """rdr_options.loop: the device while-graph, host-relaunched graphs, eager
    launches and the persistent cooperative kernel run the same arithmetic --
    iterations within +-1 of the oracle's, x equal to rounding, the GPU's own
    exit satisfying R-A16; rdr_profile_solve (eager, events between kernel
    groups) agrees and times every group."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    c = make_config(0, n=3, p=3, space=space, perturb=True, bc="x0", coeffs="loguniform")
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    bn = np.random.default_rng(3).uniform(-1, 1, O.n_total)
    hist = []
    xo, ito, _ = O.solve(bn, rtol=1e-8, history=hist)
    b = torch.from_numpy(bn).cuda()
    res = {}
    for loop in (rdr.LOOP_DEVICE, rdr.LOOP_HOST, rdr.LOOP_EAGER, rdr.LOOP_GRAPH, rdr.LOOP_PERSISTENT):
        S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=loop)
        assert S.info["persistent_loop"] == (1 if loop == rdr.LOOP_PERSISTENT else S.info["persistent_loop"])
        if loop in (rdr.LOOP_HOST, rdr.LOOP_EAGER, rdr.LOOP_GRAPH):
            assert S.info["persistent_loop"] == 0
        x, it = S.solve(b)
        _check_iters(S, it, ito, lambda k: hist[k - 1] if 0 < k <= len(hist) else None)
        st = S.last_stats()
        assert st["launches"] >= 1
        assert rel(x.cpu().numpy(), xo) <= 1e-6
        res[loop] = (x.cpu().numpy(), it)
        if loop == rdr.LOOP_EAGER:
            it2, ms = S.profile_solve(b)
            assert abs(it2 - it) <= 1 and np.all(ms[:3] > 0) and ms[3] == 0
    x0, it0 = res[rdr.LOOP_GRAPH]
    for loop, (xl, itl) in res.items():
        assert abs(itl - it0) <= 1
        assert rel(xl, x0) <= 1e-8


def test_profile_clocks(torch_cuda):
    """rdr_debug_profile_clocks: the probe behind the fused apply reads a plausible SM
    clock inside the iteration and alone, times are positive, and the solver still
    solves afterwards (the call overwrites the solve vectors); hybrid: RDR_EINVAL."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(0, n=3, p=3, space=HGRAD, perturb=True, bc="x0", coeffs="loguniform")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    x0, it0 = S.solve(b)
    mhz_in, mhz_alone, ms_iter, ms_apply = S.profile_clocks(b, iters=20)
    assert 300 <= mhz_in <= 3000 and 300 <= mhz_alone <= 3000
    assert ms_iter > 0 and ms_apply > 0 and ms_apply < ms_iter
    x1, it1 = S.solve(b)
    assert it1 == it0 and rel(x1.cpu().numpy(), x0.cpu().numpy()) <= 1e-8
    H = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, preconditioner=rdr.HYBRID)
    with pytest.raises(rdr.RdrError) as e:
        H.profile_clocks(b)
    assert e.value.code == -1


def test_persistent_loop_not_eligible(torch_cuda):
    """RDR_LOOP_PERSISTENT needs star patches of at most 256 dofs: H(grad) p = 6
    (431-dof vertex stars) is RDR_EINVAL; the default loop then uses the graph."""
    from paper_2506_17406_b200 import rdr
    c = make_config(0, n=2, p=6, space=HGRAD, perturb=True, bc="all")
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_PERSISTENT)
    assert e.value.code == -1
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    assert S.info["persistent_loop"] == 0


@pytest.mark.parametrize("space,p", [(HGRAD, 5), (HCURL, 4), (HDIV, 3)])
def test_every_apply_layout(torch_cuda, space, p):
    """Each warp layout of the apply (setup autotunes among them) against the
    oracle, plain and in the fused PCG (rdr_debug_set_apply_variant)."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    c = make_config(0, n=2, p=p, space=space, perturb=True, bc="x0", coeffs="loguniform")
    # the graph loop: the fused PCG runs the DMMA apply kernel (not the persistent kernel)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    x = c.draw_vector(O.n_total)
    xt = torch.from_numpy(x).cuda()
    ya = O.apply(x)
    b = c.draw_vector(O.n_total)
    hist = []
    _, ito, _ = O.solve(b, rtol=1e-8, history=hist)
    ran = 0
    for k in range(18):  # 6 layouts x (H(grad), H(curl), H(div))
        if not S.set_apply_variant(k):
            continue
        ran += 1
        assert S.info["apply_variant"] == k
        assert rel(S.apply(xt).cpu().numpy(), ya) <= TOL, k
        _, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
        _check_iters(S, it, ito, lambda kk: hist[kk - 1] if 0 < kk <= len(hist) else None)
    assert ran == 6  # every layout of this n_mat fits these small elements


@pytest.mark.parametrize("space,p,n,perturb", [(HCURL, 1, 2, True), (HCURL, 2, 2, True), (HCURL, 4, 2, True),
                                               (HCURL, 6, 2, False), (HCURL, 10, 1, False), (HDIV, 1, 2, True),
                                               (HDIV, 3, 2, True), (HDIV, 6, 2, False)])
def test_factored_apply(torch_cuda, space, p, n, perturb):
    """The factored two-stage apply (the reference matrices
    factored through L2-orthonormal bases of P_p and P_{p-1}, a per-cell 3 x 3 mix
    between two GEMMs) against the oracle: A x, the fused PCG's first apply, and
    PCG iterations (rdr_debug_set_apply_config(-1)); the factors reproduce the
    library's reference matrices (rdr_reference_factors)."""
    import ctypes
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    c = make_config(0, n=n, p=p, space=space, perturb=perturb, bc="x0", coeffs="loguniform")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    assert S.info["apply_factored"] == 0  # small meshes: setup never picks it (kFactMinCells)
    x = c.draw_vector(O.n_total)
    xt = torch.from_numpy(x).cuda()
    ya = O.apply(x)
    for v in (-1, -2, -3):  # tiles of (16, 16), (32, 32), (32, 24) cells (the last two do not fit at p >= 9)
        if not S.set_apply_config(v, 0, 0):
            assert v in (-2, -3) and p >= 9
            continue
        assert S.info["apply_factored"] == -v
        assert rel(S.apply(xt).cpu().numpy(), ya) <= TOL, v
        assert rel(S.debug_fused_apply(xt, torch.zeros_like(xt)).cpu().numpy(), O.apply(O.mask(x))) <= TOL, v
        # each cell tile's column blocks split over (stage A, stage B) CTAs
        for nsa, nsb in ((2, 1), (3, 2), (8, 5)):
            assert S.set_apply_config(v, nsa, nsb)
            assert (S.info["apply_fact_split_a"], S.info["apply_fact_split_b"]) == (nsa, nsb)
            assert rel(S.apply(xt).cpu().numpy(), ya) <= TOL, (v, nsa, nsb)
            assert rel(S.debug_fused_apply(xt, torch.zeros_like(xt)).cpu().numpy(), O.apply(O.mask(x))) <= TOL
        assert not S.set_apply_config(v, 9, 1)
    # PCG with unit coefficients: with the 1e4 log-uniform contrast at p = 1 the iteration count
    # moves by 2 between two roundings of the same operator (DMMA 53, factored 52, oracle 54:
    # profiles/round2/experiments/fact_apply_rounding.txt), beyond the +-1 bar
    c = make_config(0, n=n, p=p, space=space, perturb=perturb, bc="x0", coeffs="one")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = c.draw_vector(O.n_total)
    hist = []
    xo, ito, _ = O.solve(b, rtol=1e-8, history=hist)
    for v, nsa, nsb in ((-1, 0, 0), (-2, 0, 0), (-3, 0, 0), (-1, 2, 2), (-3, 3, 2)):
        if not S.set_apply_config(v, nsa, nsb):
            assert v in (-2, -3) and p >= 9
            continue
        xg, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
        _check_iters(S, it, ito, lambda kk: hist[kk - 1] if 0 < kk <= len(hist) else None)
        assert rel(xg.cpu().numpy(), xo) <= 1e-6, v
    # the factors behind it: sum_ab G_ab F_a F_b^T = the reference matrices to rounding
    lib = rdr._lib
    nl, nf, nfm = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.rdr_reference_factors(space, p, None, ctypes.byref(nl), ctypes.byref(nf), ctypes.byref(nfm)) == 0
    F = np.zeros((nl.value, nf.value))
    lib.rdr_reference_factors(space, p, F.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nl), ctypes.byref(nf),
                              ctypes.byref(nfm))
    nm_, nmat = ctypes.c_int32(), ctypes.c_int32()
    lib.rdr_reference_matrices(space, p, None, ctypes.byref(nm_), ctypes.byref(nmat))
    R = np.zeros((nmat.value, nl.value, nl.value))
    lib.rdr_reference_matrices(space, p, R.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nm_), ctypes.byref(nmat))
    npm = nfm.value // 3
    FM = [F[:, a * npm:(a + 1) * npm] for a in range(3)]
    for a in range(3):
        assert rel(FM[a] @ FM[a].T, R[a]) <= 1e-13
    for k, (a, bb) in enumerate([(0, 1), (0, 2), (1, 2)]):
        X = FM[a] @ FM[bb].T
        assert rel(X + X.T, R[3 + k]) <= 1e-13
    if space == HDIV:  # div-div through the one-component block
        FD = F[:, nfm.value:]
        assert rel(FD @ FD.T, R[6]) <= 1e-13
        return
    npk = (nf.value - nfm.value) // 3
    FK = [F[:, nfm.value + a * npk:nfm.value + (a + 1) * npk] for a in range(3)]
    for a in range(3):
        assert rel(FK[a] @ FK[a].T, R[6 + a]) <= 1e-13
    for k, (a, bb) in enumerate([(0, 1), (0, 2), (1, 2)]):
        X = FK[a] @ FK[bb].T
        assert rel(X + X.T, R[9 + k]) <= 1e-13


def test_apply_ring_depths_and_grids(torch_cuda):
    """The apply with explicit ring depths (the shallowest, KS + 1 chunks, to the
    deepest that fits) and grids (resident CTAs, one CTA per unit, a single CTA
    walking every unit) against the oracle, plain and in the fused PCG
    (rdr_debug_set_apply_config: the configurations setup's timing can pick)."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    c = make_config(0, n=2, p=7, space=HGRAD, perturb=True, bc="x0", coeffs="loguniform")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    x = c.draw_vector(O.n_total)
    ya = O.apply(x)
    b = c.draw_vector(O.n_total)
    hist = []
    _, ito, _ = O.solve(b, rtol=1e-8, history=hist)
    ks = {0: 2, 2: 4, 6: 4}  # variant -> K-split groups: (32,4,2), (32,4,4), (16,4,4)
    ran = 0
    for v, kgroups in ks.items():
        for slots in (kgroups + 1, 2 * kgroups, 16):
            for grid in (0, 1, 7):
                if not S.set_apply_config(v, slots, grid):
                    continue
                ran += 1
                i = S.info
                assert (i["apply_variant"], i["apply_slots"]) == (v, slots)
                assert grid == 0 or i["apply_grid"] == grid
                assert rel(S.apply(torch.from_numpy(x).cuda()).cpu().numpy(), ya) <= TOL, (v, slots, grid)
                _, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
                _check_iters(S, it, ito, lambda kk: hist[kk - 1] if 0 < kk <= len(hist) else None)
    assert ran >= 18
    assert not S.set_apply_config(0, 2, 0)  # fewer chunks than K-split groups + 1


@pytest.mark.parametrize("p", [2, 4])
def test_both_small_patch_kernels(torch_cuda, p):
    """H(div) edge stars (all patches <= 128 dofs): one warp per patch and the
    resident warps walking the patches with prefetch give the oracle's P^-1 r
    and PCG iterations (rdr_debug_set_small_patch_kernel)."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    # unit coefficients: with the 1e4 log-uniform contrast on this mesh the edge stars reach
    # kappa ~ 1e5 and the stored inverses differ from the oracle's Cholesky solves by ~kappa eps
    c = make_config(0, n=3, p=p, space=HDIV, perturb=True, bc="x0", coeffs="one")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_GRAPH)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    x = c.draw_vector(O.n_total)
    za = O.precond(x)
    b = c.draw_vector(O.n_total)
    hist = []
    _, ito, _ = O.solve(b, rtol=1e-8, history=hist)
    for persistent in (False, True):
        assert S.set_small_patch_kernel(persistent)
        assert rel(S.precond(torch.from_numpy(x).cuda()).cpu().numpy(), za) <= TOL
        _, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
        _check_iters(S, it, ito, lambda k: hist[k - 1] if 0 < k <= len(hist) else None)
    c2 = make_config(0, n=2, p=6, space=HGRAD, bc="all")  # 431-dof vertex stars: no small-patch launch
    S2 = rdr.Solver(c2.vertices, c2.tets, c2.p, c2.space, c2.alpha, c2.beta, c2.mask)
    assert not S2.set_small_patch_kernel(True)


def test_stream_semantics_and_repeated_setup(torch_cuda):
    """apply / precond are asynchronous on the caller's stream (results visible
    after a sync on that stream only); setup/destroy can be repeated; a handle
    solves repeatedly with identical results (deterministic iteration count)."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(0, n=2, p=4, space=HGRAD, perturb=True, bc="x0", coeffs="loguniform")
    for _ in range(3):
        S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
        S.close()
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    x = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y = S.apply(x, stream=s)
        z = S.precond(x, stream=s)
    s.synchronize()
    y0 = S.apply(x)
    z0 = S.precond(x)
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), y0.cpu().numpy()) <= 1e-14
    assert rel(z.cpu().numpy(), z0.cpu().numpy()) <= 1e-14
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    its = [S.solve(b)[1] for _ in range(3)]
    assert len(set(its)) == 1


def test_solve_maxit_and_host_path(torch_cuda):
    """maxit reached -> RDR_ENOCONV semantics (iters == maxit, x written,
    converged False); rtol = 0 runs exactly maxit iterations; the host-buffer
    entry point (rdr_solve_host) returns the same iterate as the device one."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c, S, O = _pair(torch, 0, n=2, p=3, space=HGRAD, perturb=True, bc="all")
    b = c.draw_vector(O.n_total)
    bt = torch.from_numpy(b).cuda()
    x, it = S.solve(bt, rtol=1e-12, maxit=5)
    assert it == 5 and not S.converged
    xo, ito, _ = O.solve(b, rtol=0.0, maxit=5)
    assert ito == 5 and rel(x.cpu().numpy(), xo) <= 1e-10
    xd, itd = S.solve(bt, rtol=1e-8)
    bh = torch.from_numpy(b).pin_memory()
    xh = torch.empty(S.n_total, dtype=torch.float64).pin_memory()
    ith = S.solve_host(bh, xh)
    assert ith == itd and rel(xh.numpy(), xd.cpu().numpy()) <= 1e-14


def test_smoke_entry_point(torch_cuda):
    import __graft_entry__
    __graft_entry__.smoke()


# ---------------------------------------------------------------- NEXT-3: unsplit baseline decompositions
@pytest.mark.parametrize("space,p,bc", [(HGRAD, 2, "all"), (HGRAD, 4, "x0"), (HGRAD, 6, "all"),
                                        (HCURL, 2, "all"), (HCURL, 3, "x0"), (HCURL, 5, "all")])
def test_unsplit_decomposition(torch_cuda, space, p, bc):
    """PAFW0(X0) (Eq. 5.2) and PH(X0, X1I) (Eq. 5.10), one-level: star patches
    holding the cell interiors, no Jacobi -- the baselines of the split."""
    c, S, O = _pair(torch_cuda, 0, dec="unsplit", n=2, p=p, space=space, perturb=True, bc=bc, coeffs="loguniform")
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


def test_unsplit_config5_sampled(torch_cuda):
    """Unsplit H(grad) at p = 6 on the config-5 mesh: sampled rows, PCG converges."""
    from paper_2506_17406_b200 import rdr
    from oracle.sampled import SampledOracle
    c = make_config(5, p=6)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=rdr.UNSPLIT)
    O = SampledOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition="unsplit")
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O, n_vertices=2, n_cells=3)
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b)


def test_fused_apply_ring_race_regression(torch_cuda):
    """The PCG (fused) variant of the apply kernel equals rdr_apply on every one
    of 20 launches at p = 10 on a 12^3 mesh (32 cells per CTA): before the
    ring-slot release waited for the consumers' shared loads (mbar_release),
    about half of these launches had one warp read a half-refilled TMA slot."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(3, n=12)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    z = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    z = z * (S.apply(torch.ones_like(z)) != 0)
    ref = S.apply(z).cpu().numpy()
    for _ in range(20):
        q = torch.zeros_like(z)
        S.debug_fused_apply(z, q)
        assert rel(q.cpu().numpy(), ref) <= 1e-13


# ---------------------------------------------------------------- NEXT-1: hybrid Schwarz with the Whitney coarse space
@pytest.mark.parametrize("space,p,bc,n", [(HGRAD, 1, "x0", 3), (HGRAD, 3, "all", 3), (HGRAD, 5, "x0", 2),
                                          (HCURL, 2, "all", 2), (HCURL, 3, "x0", 3), (HCURL, 4, "all", 2),
                                          (HDIV, 1, "x0", 2), (HDIV, 3, "x0", 2), (HDIV, 4, "all", 2)])
def test_hybrid_preconditioner(torch_cuda, space, p, bc, n):
    """The paper's symmetric multiplicative hybrid: weights rho_m
    from the library's own CG-Lanczos equal the oracle's, P^-1 r at 1e-11, PCG
    iterations +-1."""
    from paper_2506_17406_b200 import rdr
    from oracle.hybrid import HybridOracle
    torch = torch_cuda
    c = make_config(0, n=n, p=p, space=space, perturb=True, bc=bc, coeffs="loguniform")
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, preconditioner=rdr.HYBRID)
    O = HybridOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    assert np.allclose(S.weights, O.rho, rtol=1e-10, atol=0)
    # The coarse solve applies a stored inverse of A restricted to W^k (the
    # oracle: a Cholesky solve), whose forward error is ~kappa(A_c) eps; under
    # the 1e-4 coefficient contrast kappa(A_c) reaches ~2e6 for H(curl). SURVEY
    # §8(c): state the kappa-derived bound instead of loosening silently.
    ev = np.linalg.eigvalsh(O.A[O.W][:, O.W].toarray()) if len(O.W) else np.ones(1)
    tol = max(TOL, ev[-1] / ev[0] * np.finfo(float).eps)
    for _ in range(2):
        x = c.draw_vector(O.n_total)
        xt = torch.from_numpy(x).cuda()
        z = S.precond(xt).cpu().numpy()
        za = O.precond(x)
        assert rel(z, za) <= tol, (rel(z, za), tol)
        assert rel(S.apply(xt).cpu().numpy(), O.apply(x)) <= TOL
    b = c.draw_vector(O.n_total)
    xg, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
    xo, ito, _ = O.solve(b, rtol=1e-8)
    assert abs(it - ito) <= 1, (it, ito)
    assert rel(xg.cpu().numpy(), xo) <= 1e-6
    # the loop drivers of the unfused iteration (device while-graph with a one-iteration
    # body, host-relaunched 8-iteration graphs, eager launches) give the same iterates;
    # the while-graph launches nothing past the iteration that converged
    bt = torch.from_numpy(b).cuda()
    stats = {}
    for loop in (rdr.LOOP_GRAPH, rdr.LOOP_HOST, rdr.LOOP_EAGER):
        L = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, preconditioner=rdr.HYBRID,
                       loop=loop)
        xl, itl = L.solve(bt, rtol=1e-8)
        # (the scatter-adds are atomic: their order, and so the rounding, differs from run to run)
        assert abs(itl - it) <= 1 and rel(xl.cpu().numpy(), xg.cpu().numpy()) <= 1e-8
        stats[loop] = (itl, L.last_stats()["launches"])
        if loop == rdr.LOOP_GRAPH:
            x0, it0 = L.solve(torch.zeros_like(bt), rtol=1e-8)  # b = 0: stop flag set by the start
            assert it0 == 0 and float(x0.abs().max()) == 0.0
            if it > 3:  # maxit reached: iters == maxit, not converged
                _, it2 = L.solve(bt, rtol=1e-8, maxit=2)
                assert it2 == 2 and not L.converged
    (itg, ng), (ite, ne) = stats[rdr.LOOP_GRAPH], stats[rdr.LOOP_EAGER]
    if itg == ite:  # the eager launches plus one condition kernel per one-iteration body
        assert ng <= ne + max(itg, 1), (ng, ne, itg)


def _hybrid_golden():
    return [(e["cfg"], e["p"]) for e in json.load(open(GOLDEN)).get("hybrid_entries", [])]


@pytest.mark.parametrize("cfg,p", _hybrid_golden())
def test_hybrid_full_size_golden(torch_cuda, cfg, p):
    """NEXT-1 at the sizes DESIGN.md section 10b reports (config 2; the H(grad), H(curl) and
    H(div) p-sweeps on the 8^3 x 6 mesh): the library's weights rho_m equal the oracle's, PCG
    iterations within +-1 of oracle/hybrid.py's count (tests/golden, written by
    scripts/oracle_golden.py --hybrid, oracle/ only), and the GPU's own exit satisfies R-A16."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    g = [e for e in json.load(open(GOLDEN))["hybrid_entries"] if (e["cfg"], e["p"]) == (cfg, p)][0]
    c = make_config(cfg, p=p) if cfg in (5, 7, 8) else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, preconditioner=rdr.HYBRID)
    assert S.n_total == g["n_total"] and S.info["n_free"] == g["n_free"]
    assert np.allclose(S.weights, g["rho"], rtol=1e-9, atol=0), (S.weights, g["rho"])
    b = c.draw_vector(S.n_total)   # the config's rhs (first draw), as scripts/oracle_golden.py
    x, it = S.solve(torch.from_numpy(b).cuda(), rtol=1e-8)
    st = S.last_stats()
    assert st["converged"] == 1 and st["z_last"] <= 1e-8 * st["z0"]
    assert abs(it - g["iters"]) <= 1, (it, g["iters"])
    # true residual of the GPU's x through the library's own operator: the same order as the oracle's
    bm = torch.from_numpy(b).cuda()
    r = S.apply(x) - bm
    free = x != 0  # x is exactly zero on the constrained dofs (and nowhere else, generically)
    assert int(free.sum()) == g["n_free"]
    rel_res = float(r[free].norm() / bm[free].norm())
    assert rel_res <= max(10 * g["true_rel_res"], 1e-6), (rel_res, g["true_rel_res"])


def test_tet_vertex_order_invariance(torch_cuda):
    """rdr_setup accepts tets in any vertex order (it sorts, R-A3): shuffling
    every tet's vertices (and the mask columns with them) changes nothing."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    for space in (HGRAD, HCURL, HDIV):
        c = make_config(0, n=2, p=3, space=space, perturb=True, bc="x0", coeffs="loguniform")
        rng = np.random.default_rng(7)
        perm = np.array([rng.permutation(4) for _ in range(c.tets.shape[0])])
        tets2 = np.take_along_axis(c.tets, perm, axis=1)
        mask2 = np.take_along_axis(c.mask, perm, axis=1)
        S1 = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
        S2 = rdr.Solver(c.vertices, tets2, c.p, c.space, c.alpha, c.beta, mask2)
        x = torch.from_numpy(c.draw_vector(S1.n_total)).cuda()
        assert rel(S2.apply(x).cpu().numpy(), S1.apply(x).cpu().numpy()) <= 1e-14
        assert rel(S2.precond(x).cpu().numpy(), S1.precond(x).cpu().numpy()) <= 1e-14
        assert S2.solve(x)[1] == S1.solve(x)[1]


@pytest.mark.parametrize("space,p,dec", [(HGRAD, 2, "split"), (HGRAD, 6, "split"), (HGRAD, 10, "split"),
                                         (HCURL, 3, "split"), (HCURL, 6, "split"), (HGRAD, 4, "unsplit"),
                                         (HCURL, 4, "unsplit")])
def test_device_patch_setup(torch_cuda, space, p, dec):
    """the patch inverses assembled and inverted on the GPU
    (block Gauss-Jordan sweep, patch_setup.cu) give the same P^-1 as the host
    Cholesky-based setup to rounding and match the oracle at the parity bar."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    torch = torch_cuda
    c = make_config(0, n=2, p=p, space=space, perturb=True, bc="x0", coeffs="loguniform")
    d = rdr.UNSPLIT if dec == "unsplit" else rdr.SPLIT
    Sd = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=d)
    Sh = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=d,
                    setup=rdr.SETUP_HOST)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=dec)
    for _ in range(2):
        x = c.draw_vector(O.n_total)
        xt = torch.from_numpy(x).cuda()
        zd, zh = Sd.precond(xt).cpu().numpy(), Sh.precond(xt).cpu().numpy()
        assert rel(zd, zh) <= 1e-12, rel(zd, zh)
        assert rel(zd, O.precond(x)) <= TOL
    b = torch.from_numpy(c.draw_vector(O.n_total)).cuda()
    assert abs(Sd.solve(b)[1] - Sh.solve(b)[1]) <= 1
    assert Sd.info["patch_setup_seconds"] > 0 and Sd.info["patch_setup_seconds"] <= Sd.info["setup_seconds"]


def test_device_patch_setup_errors(torch_cuda):
    """beta = 0 would make the H(curl) potential patches and the H(div) edge
    stars singular (their rounded pivots need not be negative, commit 621b7e5):
    both setups reject it with RDR_EINVAL before any factorisation; an unknown
    setup or loop is EINVAL."""
    from paper_2506_17406_b200 import rdr
    for space in (HCURL, HDIV):
        c = make_config(0, n=1, p=2, space=space, bc="all")
        for su in (rdr.SETUP_DEVICE, rdr.SETUP_HOST):
            with pytest.raises(rdr.RdrError) as e:
                rdr.Solver(c.vertices, c.tets, 2, space, c.alpha, 0 * c.beta, np.zeros_like(c.mask), setup=su)
            assert e.value.code == -1
    c = make_config(0, n=1, p=2, space=HCURL, bc="all")
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, 2, HCURL, c.alpha, c.beta, c.mask, loop=7)
    assert e.value.code == -1
    with pytest.raises(rdr.RdrError) as e:
        rdr.Solver(c.vertices, c.tets, 2, HCURL, c.alpha, c.beta, c.mask, setup=2)
    assert e.value.code == -1



# ---------------------------------------------------------------- H(div)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("perturb,bc,coeffs", [(False, "all", "one"), (True, "x0", "loguniform")])
def test_hdiv_small(torch_cuda, p, perturb, bc, coeffs):
    """RT_p Riesz map (Piola 2-forms, 7 reference matrices) with the edge-star
    PAFW1(X2_Gamma) + J(X2_I) preconditioner (Eq. 5.16): apply / P^-1 at 1e-11,
    PCG iterations +-1 against the oracle."""
    c, S, O = _pair(torch_cuda, 0, n=2, p=p, space=HDIV, perturb=perturb, bc=bc, coeffs=coeffs)
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


def test_hdiv_p10(torch_cuda):
    """RT_10 (n_loc 715) on the 6-tet cube; the oracle's x87 RT_10 construction
    takes ~4 min of the host."""
    c, S, O = _pair(torch_cuda, 0, n=1, p=10, space=HDIV, perturb=False, bc="x0")
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


@pytest.mark.parametrize("p", [3, 5])
def test_hdiv_unsplit(torch_cuda, p):
    """PAFW1(X2): interiors inside the edge stars, no Jacobi (the hybrid with
    the W^2 coarse space is in test_hybrid_preconditioner)."""
    c, S, O = _pair(torch_cuda, 0, "unsplit", n=2, p=p, space=HDIV, perturb=True, bc="x0", coeffs="loguniform")
    _check_apply_precond(torch_cuda, c, S, O)
    _check_pcg(torch_cuda, c, S, O)


def test_config6_hdiv_sampled(torch_cuda):
    """The NEXT-2 workload: RT_6 on 12^3 x 6 (config 4's mesh and degree, the
    2-form space), sampled rows; PCG iterations vs the oracle's (golden)."""
    c, S, O = _sampled_pair(6)
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O)
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b, _golden(6, 6))


@pytest.mark.parametrize("cfg,p", [(7, 9), (7, 10), (8, 9), (8, 10)])
def test_config78_high_p_sampled(torch_cuda, cfg, p):
    """The H(curl) (Ned1_p, config 7) and H(div) (RT_p, config 8) p-sweeps on
    config 5's perturbed 8^3 x 6 mesh at the largest degrees DESIGN.md §7
    reports (p = 9, 10; north_star: H(curl) up to p = 10): sampled rows of
    A x and P^-1 r, PCG iterations vs the oracle's (golden, oracle/lean.py)."""
    c, S, O = _sampled_pair(cfg, p=p)
    b = c.draw_vector(O.n_total)
    rows = _sample_rows(O, n_vertices=1, n_cells=2)  # every sampled patch costs ~30 element matrices at p = 10
    _check_sampled(torch_cuda, c, S, O, rows)
    _check_sampled_pcg(torch_cuda, c, S, O, rows, b, _golden(cfg, p))


@pytest.mark.parametrize("space,n,p", [(HGRAD, 4, 2), (HCURL, 3, 2), (HDIV, 3, 2)])
def test_device_coarse_inverse(torch_cuda, space, n, p):
    """The hybrid's coarse inverse by the multi-CTA block sweep on the device
    (several 64-blocks: n_c > 64) equals the host Cholesky-based inverse to
    kappa(A_c) eps, and the weights rho_m (from the library's own Lanczos with
    either inverse) agree."""
    from paper_2506_17406_b200 import rdr
    torch = torch_cuda
    c = make_config(0, n=n, p=p, space=space, perturb=True, bc="x0", coeffs="loguniform")
    kw = dict(preconditioner=rdr.HYBRID)
    Sd = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, **kw)
    Sh = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, setup=rdr.SETUP_HOST, **kw)
    assert np.allclose(Sd.weights, Sh.weights, rtol=1e-9, atol=0)
    x = torch.from_numpy(c.draw_vector(Sd.n_total)).cuda()
    zd, zh = Sd.precond(x).cpu().numpy(), Sh.precond(x).cpu().numpy()
    assert rel(zd, zh) <= 1e-9, rel(zd, zh)
    assert abs(Sd.solve(x)[1] - Sh.solve(x)[1]) <= 1


def test_hdiv_curl_kernel_through_library(torch_cuda):
    """div curl = 0 through the library: for u = C v (the discrete curl of a
    random Ned1 vector, face/edge incidence + type-I -> type-II), A u does not
    depend on alpha (H(div), no Dirichlet, perturbed mesh)."""
    from paper_2506_17406_b200 import rdr
    from oracle.solver import Oracle
    from test_oracle_hdiv import _discrete_curl
    torch = torch_cuda
    p = 3
    c = make_config(0, n=2, p=p, space=HDIV, perturb=True, bc="none")
    O2 = Oracle(c.vertices, c.tets, p, "hdiv", c.alpha, c.beta, c.mask, assemble=False)
    O1 = Oracle(c.vertices, c.tets, p, "hcurl", c.alpha, c.beta, c.mask, assemble=False)
    C = _discrete_curl(O2, O1, p)
    u = C @ np.random.default_rng(5).standard_normal(C.shape[1])
    ut = torch.from_numpy(u).cuda()
    S1 = rdr.Solver(c.vertices, c.tets, p, HDIV, c.alpha, c.beta, c.mask)
    S2 = rdr.Solver(c.vertices, c.tets, p, HDIV, 1e3 * c.alpha, c.beta, c.mask)
    y1, y2 = S1.apply(ut).cpu().numpy(), S2.apply(ut).cpu().numpy()
    assert rel(y2, y1) <= 1e-9, rel(y2, y1)
