"""Pins of the memory-lean oracle (oracle/lean.py) against the global oracle
(oracle/solver.py, itself pinned by test_oracle_*.py): the same operator,
preconditioner and PCG iterates on small meshes of every space, perturbed,
partial Dirichlet and log-uniform coefficients (SURVEY §8(c) config-3 scope)."""
import numpy as np
import pytest

from rdr_inputs import make_config, HGRAD, HCURL, HDIV
from oracle.solver import Oracle
from oracle.lean import LeanOracle


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("space,p,bc,coeffs", [
    (HGRAD, 4, "all", "one"), (HGRAD, 3, "x0", "loguniform"),
    (HCURL, 3, "all", "one"), (HCURL, 2, "x0", "loguniform"),
    (HDIV, 3, "all", "one"), (HDIV, 2, "x0", "loguniform")])
def test_lean_equals_global(space, p, bc, coeffs, tmp_path):
    c = make_config(0, n=2, p=p, space=space, perturb=True, bc=bc, coeffs=coeffs)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    L = LeanOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask,
                   store_dir=str(tmp_path) if space == HCURL else None)
    O.build_preconditioner(kappa=False)
    L.build_preconditioner()
    assert len(L.factors) == len(O.factors)
    for _ in range(2):
        x = c.draw_vector(O.n_total)
        assert rel(L.apply(x), O.apply(x)) <= 1e-13
        assert rel(L.precond(x), O.precond(x)) <= 1e-12
        assert np.all(L.apply(x)[~O.free] == 0) and np.all(L.precond(x)[~O.free] == 0)
    b = c.draw_vector(O.n_total)
    ho, hl = [], []
    xo, ito, _ = O.solve(b, rtol=1e-8, history=ho)
    xl, itl, _ = L.solve(b, rtol=1e-8, history=hl)
    assert itl == ito
    assert rel(xl, xo) <= 1e-10
    # rounding differences grow along the Krylov sequence (to percent level at the
    # end for the 1e4 coefficient contrast): compare the first 20 iterates
    np.testing.assert_allclose(hl[:20], ho[:20], rtol=1e-6)
