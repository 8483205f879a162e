"""The paper's symmetric hybrid Schwarz preconditioner with the Whitney coarse
space.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:2399-2455: the subspaces of the split decompositions (Eq. 5.4 / 5.12 plus W^k)
  X_1 = X_I (interior dofs, point-Jacobi),
  X_2 = X_Gamma (interface, the additive star-patch solver of oracle.solver),
  X_3 = W^k (lowest order: the vertex dofs for H(grad), the Whitney edge dofs
        for H(curl) -- Lemma 4.1, makes W^k a column selection),
each with the inexact solver rho_m a~_m, "combined multiplicatively from
right to left to right for symmetry": the sweep X_1, X_2, X_3, X_2, X_1.
rho_m = (lambda~_min + 3 lambda~_max) / 4 with lambda~ the extreme eigenvalues
of a(u, v) = lambda a~_m(u, v) on X_m, "computed from 10 conjugate gradient
iterations with a randomized right hand side" (Lanczos).
Readings (DESIGN.md R-N1..N3): the paper's W^k solver is a GMG V-cycle with a
coarse Cholesky; here it is an exact solve on W^k of the given mesh (the
configs are single-level meshes). The random rhs is the counter-based
uniform[-1,1] vector `lanczos_rhs` (splitmix64), restricted to X_m. The exact
coarse solver has rho_3 = 1.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .solver import Oracle

LANCZOS_STEPS = 10
LANCZOS_SEED = 0x5EED


def lanczos_rhs(n: int, seed: int = LANCZOS_SEED) -> np.ndarray:
    """uniform[-1,1] from splitmix64(seed + i) (53 high bits), i = 0..n-1."""
    with np.errstate(over="ignore"):
        z = (np.arange(n, dtype=np.uint64) + np.uint64(seed)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def cg_lanczos_extremes(apply_A, apply_P, b, steps=LANCZOS_STEPS):
    """Extreme eigenvalues of P A (P the inexact solver's inverse) on the
    subspace of b, from the Lanczos tridiagonal of `steps` PCG iterations."""
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_P(r)
    p = z.copy()
    rz = r @ z
    alphas, betas = [], []
    for _ in range(steps):
        if rz <= 0:
            break
        q = apply_A(p)
        a = rz / (p @ q)
        alphas.append(a)
        x += a * p
        r -= a * q
        z = apply_P(r)
        rz_new = r @ z
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    k = len(alphas)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(betas[j]) / alphas[j]
    ev = np.linalg.eigvalsh(T)
    return ev[0], ev[-1]


class HybridOracle(Oracle):
    """Oracle with the symmetric multiplicative hybrid preconditioner."""

    def __init__(self, vertices, tets, p, space, alpha, beta, mask):
        super().__init__(vertices, tets, p, space, alpha, beta, mask)
        self.build_preconditioner(kappa=False)
        num = self.num
        fr = self.free
        self.I = np.nonzero(num.interior & fr)[0]                       # X_1
        self.Gam = np.nonzero(~num.interior & fr)[0]                    # X_2
        if self.space == "hgrad":                                       # X_3 = W^0: vertex dofs
            w = np.arange(num.offsets[0], num.offsets[0] + self.topo.nv)
        elif self.space == "hcurl":                                     # X_3 = W^1: Whitney edge dofs
            w = num.offsets[1] + np.arange(self.topo.ne) * num.per[1]
        else:                                                           # X_3 = W^2: Whitney face dofs
            w = num.offsets[2] + np.arange(self.topo.nf) * num.per[2]
        self.W = w[fr[w]]
        Ac = self.A[self.W][:, self.W].toarray()
        self.coarse = sla.cho_factor(Ac, lower=True) if len(self.W) else None
        self.rho = [self._rho(self.I, self._solve_jacobi), self._rho(self.Gam, self._solve_patches), 1.0]

    # the three inexact solvers, each returning a full-length correction
    def _solve_jacobi(self, r):
        z = np.zeros_like(r)
        z[self.int_idx] = self.dinv * r[self.int_idx]
        return z

    def _solve_patches(self, r):
        z = np.zeros_like(r)
        for kind, idx, emb, fac in self.factors:
            if kind == "dof":
                z[idx] += sla.cho_solve(fac, r[idx])
            else:
                z += emb @ sla.cho_solve(fac, emb.T @ r)
        z[~self.free] = 0.0
        return z

    def _solve_coarse(self, r):
        z = np.zeros_like(r)
        if self.coarse is not None:
            z[self.W] = sla.cho_solve(self.coarse, r[self.W])
        return z

    def _rho(self, sub, solver):
        """rho_m = (lambda_min + 3 lambda_max) / 4 of solver^-1 A restricted to X_m."""
        if len(sub) == 0:
            return 1.0
        mask = np.zeros(self.n_total)
        mask[sub] = 1.0
        b = lanczos_rhs(self.n_total) * mask
        lo, hi = cg_lanczos_extremes(lambda v: mask * (self.A @ (mask * v)), lambda v: mask * solver(mask * v), b)
        return (lo + 3.0 * hi) / 4.0

    def precond(self, r):
        """Symmetric multiplicative sweep X_1, X_2, X_3, X_2, X_1 with the damped
        solvers (1/rho_m) a~_m^-1."""
        r = self.mask(r)
        stages = [(self._solve_jacobi, self.rho[0]), (self._solve_patches, self.rho[1]), (self._solve_coarse, self.rho[2]),
                  (self._solve_patches, self.rho[1]), (self._solve_jacobi, self.rho[0])]
        e = np.zeros_like(r)
        for k, (solver, rho) in enumerate(stages):
            res = r if k == 0 else r - self.A @ e
            e += solver(res) / rho
        e[~self.free] = 0.0
        return e
