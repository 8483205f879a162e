"""The sampled-row oracle (oracle/sampled.py, used for full-size parity at
configs 3-5) against the global oracle: same rows of A x and P^-1 r on small
meshes, both spaces, partial Dirichlet and coefficient contrast."""
import numpy as np
import pytest

from rdr_inputs import make_config, HGRAD, HCURL
from oracle.solver import Oracle
from oracle.sampled import SampledOracle


@pytest.mark.parametrize("dec", ["split", "unsplit"])
@pytest.mark.parametrize("space,p,bc,coeffs", [(HGRAD, 3, "all", "one"), (HGRAD, 4, "x0", "loguniform"),
                                                (HCURL, 2, "all", "one"), (HCURL, 4, "x0", "loguniform")])
def test_sampled_rows_match_global(space, p, bc, coeffs, dec):
    c = make_config(0, n=2, p=p, space=space, perturb=True, bc=bc, coeffs=coeffs)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=dec)
    S = SampledOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, decomposition=dec)
    x = c.draw_vector(O.n_total)
    rng = np.random.default_rng(5)
    # every dof kind: vertex/edge/face/cell entities, constrained and free
    rows = np.unique(np.concatenate([rng.choice(O.n_total, 40, replace=False),
                                     [O.num.offsets[d] for d in range(4) if O.num.per[d]]]))
    y, z = O.apply(x), O.precond(x)
    ys, zs = S.apply_rows(x, rows), S.precond_rows(x, rows)
    assert np.allclose(ys, y[rows], rtol=1e-12, atol=1e-12 * np.abs(y).max())
    assert np.allclose(zs, z[rows], rtol=1e-12, atol=1e-12 * np.abs(z).max())


def test_precond_residual_rows():
    """P^-1 (b - A x) on sampled rows equals the global oracle's, at an
    arbitrary x (so the stopping-rule check of the full-size tests is exact)."""
    c = make_config(0, n=2, p=3, space=HCURL, perturb=True, bc="x0", coeffs="loguniform")
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    S = SampledOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b, x = c.draw_vector(O.n_total), c.draw_vector(O.n_total)
    rows = np.random.default_rng(2).choice(O.n_total, 30, replace=False)
    ref = O.precond(O.mask(b) - O.apply(x))[rows]
    got = S.precond_residual_rows(b, x, rows)
    assert np.allclose(got, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
