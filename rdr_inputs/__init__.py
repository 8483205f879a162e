"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method: it only generates meshes,
coefficients, Dirichlet masks and random vectors with the shapes and
distributions of the paper's Riesz-map experiments (§6.1,
P:2313-2328: Freudenthal cube meshes, random right-hand side, rtol 1e-8) as
fixed by BASELINE.json `configs` and SURVEY.md §8(d) "Input generator".

Both the oracle (oracle/) and the CUDA path (paper_2506_17406_b200/) consume
these arrays; neither imports the other.

RNG contract: rng = numpy.random.default_rng(seed); draws in
this order, each only if the config needs it:
  1. D = rng.uniform(-0.2h, 0.2h, (nv, 3)), applied to interior vertices only;
  2. log10(alpha) = rng.uniform(-2, 2, nt);
  3. log10(beta)  = rng.uniform(-2, 2, nt);
  4. b = rng.uniform(-1, 1, N_total)  (constrained entries are zeroed by the consumer);
  5. x_test = rng.uniform(-1, 1, N_total).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

HGRAD = 0
HCURL = 1
HDIV = 2

# Freudenthal/Kuhn split of a cube into 6 tets: local corners
# v0..v7 with bit0=+x, bit1=+y, bit2=+z.
_KUHN = ((0, 1, 3, 7), (0, 2, 3, 7), (0, 1, 5, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7))


def freudenthal(n: int):
    """Unit cube split into n^3 subcubes x 6 tets.

    Vertex (i,j,k)/n has id i + (n+1)(j + (n+1)k); cubes are visited
    x-fastest, then y, then z. Returns (vertices float64 [nv,3],
    tets int32 [nt,4], lattice int64 [nv,3]).
    """
    m = n + 1
    idx = np.arange(m)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    lattice = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.int64)
    vertices = lattice.astype(np.float64) / n
    tets = []
    for cz in range(n):
        for cy in range(n):
            for cx in range(n):
                corner = []
                for c in range(8):
                    di, dj, dk = c & 1, (c >> 1) & 1, (c >> 2) & 1
                    corner.append((cx + di) + m * ((cy + dj) + m * (cz + dk)))
                for t in _KUHN:
                    tets.append([corner[a] for a in t])
    return vertices, np.asarray(tets, dtype=np.int32), lattice


def boundary_mask(tets: np.ndarray, lattice: np.ndarray, n: int, kind: str) -> np.ndarray:
    """uint8 [nt,4]: bit (t,i)=1 iff the face opposite input vertex i of tet t
    lies on the requested part of the cube boundary.

    kind: "all" (whole boundary), "x0" (the x=0 face), "none".
    Decided on the integer lattice, so it is exact for perturbed meshes too
    (boundary vertices are never moved).
    """
    nt = tets.shape[0]
    mask = np.zeros((nt, 4), dtype=np.uint8)
    if kind == "none":
        return mask
    for i in range(4):
        face = np.delete(tets, i, axis=1)  # [nt,3]
        L = lattice[face]  # [nt,3,3]
        on = np.zeros(nt, dtype=bool)
        for d in range(3):
            for val in (0, n):
                if kind == "x0" and not (d == 0 and val == 0):
                    continue
                on |= np.all(L[:, :, d] == val, axis=1)
        mask[:, i] = on
    return mask


@dataclass
class Config:
    """One BASELINE.json configuration."""
    name: str
    space: int
    p: int
    n: int
    vertices: np.ndarray
    tets: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    mask: np.ndarray
    rng: np.random.Generator = field(repr=False)
    lattice: np.ndarray = field(repr=False, default=None)

    def draw_vector(self, n_total: int) -> np.ndarray:
        """Next uniform[-1,1] vector of length n_total from the config's stream
        (rhs first, then test vectors). Constrained entries are NOT zeroed here."""
        return self.rng.uniform(-1.0, 1.0, n_total)


def make_mesh(n: int, perturb: bool, rng: np.random.Generator):
    vertices, tets, lattice = freudenthal(n)
    if perturb:
        h = 1.0 / n
        D = rng.uniform(-0.2 * h, 0.2 * h, (vertices.shape[0], 3))
        interior = np.all((lattice > 0) & (lattice < n), axis=1)
        vertices = vertices.copy()
        vertices[interior] += D[interior]
    return vertices, tets, lattice


def make_config(cfg: int, p: int | None = None, seed: int = 0, n: int | None = None,
                space: int | None = None, perturb: bool | None = None,
                bc: str | None = None, coeffs: str | None = None) -> Config:
    """BASELINE.json configs[cfg-1] (1-based ids as in SURVEY §8(d)).

    1: H(grad) p=3, 2^3, unperturbed, alpha=beta=1, full Dirichlet.
    2: H(grad) p=6, 8^3, perturbed, log-uniform alpha,beta in [1e-2,1e2], Dirichlet x=0.
    3: H(grad) p=10, 16^3, perturbed, alpha=beta=1, full Dirichlet.
    4: H(curl) Ned1_6, 12^3, unperturbed, alpha=beta=1, full tangential Dirichlet.
    5: H(grad) p in 1..12 (argument p), 8^3, perturbed, alpha=beta=1, full Dirichlet.
    6: H(div) RT_6, 12^3, unperturbed, alpha=beta=1, full normal Dirichlet -- NOT a
       BASELINE.json config: the SURVEY NEXT-2 workload, config 4's mesh and degree
       with the 2-form space (PAFW1(X2_Gamma) + J(X2_I)).
    7, 8: config 5's p-sweep mesh (8^3, perturbed, alpha=beta=1, full Dirichlet) with
       H(curl) Ned1_p and H(div) RT_p, p in 1..10 -- NOT BASELINE.json configs (measurement
       of the p-robustness the paper claims for all three splits).
    0: custom small case (all of n, p, space, perturb, bc, coeffs given).
    Any keyword overrides the config's default (used for small parity meshes).
    """
    table = {
        1: dict(space=HGRAD, p=3, n=2, perturb=False, bc="all", coeffs="one"),
        2: dict(space=HGRAD, p=6, n=8, perturb=True, bc="x0", coeffs="loguniform"),
        3: dict(space=HGRAD, p=10, n=16, perturb=True, bc="all", coeffs="one"),
        4: dict(space=HCURL, p=6, n=12, perturb=False, bc="all", coeffs="one"),
        5: dict(space=HGRAD, p=6, n=8, perturb=True, bc="all", coeffs="one"),
        6: dict(space=HDIV, p=6, n=12, perturb=False, bc="all", coeffs="one"),
        7: dict(space=HCURL, p=6, n=8, perturb=True, bc="all", coeffs="one"),
        8: dict(space=HDIV, p=6, n=8, perturb=True, bc="all", coeffs="one"),
        0: dict(space=HGRAD, p=2, n=2, perturb=False, bc="all", coeffs="one"),
    }
    d = dict(table[cfg])
    for k, v in dict(p=p, n=n, space=space, perturb=perturb, bc=bc, coeffs=coeffs).items():
        if v is not None:
            d[k] = v
    rng = np.random.default_rng(seed)
    vertices, tets, lattice = make_mesh(d["n"], d["perturb"], rng)
    nt = tets.shape[0]
    if d["coeffs"] == "loguniform":
        alpha = 10.0 ** rng.uniform(-2.0, 2.0, nt)
        beta = 10.0 ** rng.uniform(-2.0, 2.0, nt)
    elif d["coeffs"] == "one":
        alpha = np.ones(nt)
        beta = np.ones(nt)
    else:
        raise ValueError(d["coeffs"])
    mask = boundary_mask(tets, lattice, d["n"], d["bc"])
    return Config(name=f"cfg{cfg}", space=d["space"], p=d["p"], n=d["n"], vertices=vertices,
                  tets=tets, alpha=alpha, beta=beta, mask=mask, rng=rng, lattice=lattice)
