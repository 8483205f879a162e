"""Quadrature and physical-space assembly of the Riesz-map operator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

a^k(u, v) = (u, beta v) + (d^k u, alpha d^k v)   (Eq. 2.9)
with the pullbacks of Eq. 2.7: k=0: phi = phi-hat o F^-1,
grad phi = J^-T grad-hat phi-hat; k=1: phi = J^-T phi-hat,
curl phi = J curl-hat phi-hat / det J; k=2: phi = J phi-hat / det J,
div phi = div-hat phi-hat / det J. Element matrices are computed by
quadrature at physical points (collapsed Gauss-Jacobi, exact to degree
2p+2, DESIGN.md R-A10), never by the reference-matrix contraction the GPU
path uses. Global CSR by the canonical numbering; Dirichlet by elimination.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np
import scipy.sparse as sp
from scipy.special import roots_jacobi

from .refelem import element, tabulate
from .simplex import reference_tet


def gauss_jacobi01(m: int, a: float):
    """m-point Gauss rule on [0,1] for weight (1-u)^a."""
    x, w = roots_jacobi(m, a, 0.0)
    return (1 + x) / 2, w / 2 ** (a + 1)


def tet_quadrature(degree: int):
    """Stroud conical product rule on the tet, exact for polynomials of total
    degree <= `degree`. Returns barycentric points [nq,4] and weights summing
    to 1 (so int_T f = |T| sum_q w_q f(x_q))."""
    m = degree // 2 + 1
    u, wu = gauss_jacobi01(m, 2.0)
    v, wv = gauss_jacobi01(m, 1.0)
    w, ww = gauss_jacobi01(m, 0.0)
    U, V, W = np.meshgrid(u, v, w, indexing="ij")
    WT = (wu[:, None, None] * wv[None, :, None] * ww[None, None, :])
    xi = U
    eta = (1 - U) * V
    zeta = (1 - U) * (1 - V) * W
    lam = np.stack([1 - xi - eta - zeta, xi, eta, zeta], axis=-1).reshape(-1, 4)
    wts = WT.reshape(-1) * 6.0
    return lam, wts


@lru_cache(maxsize=None)
def _tabulation(space: str, p: int):
    """Quadrature exact to degree 2p+2 (R-A10) and the reference basis values /
    derivatives at its points, tabulated in extended precision and rounded once;
    computed once per (space, p) and process (read-only arrays)."""
    lam, w = tet_quadrature(2 * p + 2)
    val, der = tabulate(element(space, p), lam.astype(np.longdouble))
    out = (lam, w, val.astype(np.float64), der.astype(np.float64))
    for a in out:
        a.setflags(write=False)
    return out


class Assembler:
    def __init__(self, space: str, p: int, topo, numbering):
        self.space, self.p = space, p
        self.topo, self.num = topo, numbering
        self.el = element(space, p)
        self.lam, self.w, self.val, self.der = _tabulation(space, p)
        T = reference_tet()
        self.Vhat = T.coords.astype(np.float64)
        self.Ehat_inv = np.linalg.inv((self.Vhat[1:] - self.Vhat[0]).T)
        self.vol_hat = float(T.vol)

    def jacobians(self, cells):
        x = self.topo.vertices[self.topo.cells[cells]]        # [nc,4,3] sorted order
        E = np.transpose(x[:, 1:] - x[:, :1], (0, 2, 1))       # columns x_k - x_0
        return E @ self.Ehat_inv                              # J with F(V-hat_k) = x_k

    def _weighted(self, which):
        """sqrt(w_q) R[q, n, :] of the tabulated values ("val") or derivatives
        ("der"), stored [n, q, b] (b = the reference frame components) so that
        the physical quantities below come out as [cells, n, q*3] rows."""
        key = "_w_" + which
        if not hasattr(self, key):
            R = getattr(self, which)
            sw = np.sqrt(self.w)
            Rw = R * (sw[:, None, None] if R.ndim == 3 else sw[:, None])
            setattr(self, key, np.ascontiguousarray(np.swapaxes(Rw, 0, 1)))
        return getattr(self, key)

    @staticmethod
    def _gram_phys(Jm, Rw, det=None):
        """sum_q w_q F_c(x_q)_i . F_c(x_q)_j for F_c = Jm_c R(x_q) (/ det_c): the
        physical vector field of every basis function at every quadrature point
        of cell c, contracted over points and Cartesian components."""
        nc, n, nq = Jm.shape[0], Rw.shape[0], Rw.shape[1]
        F = np.matmul(Rw.reshape(1, n * nq, 3), np.transpose(Jm, (0, 2, 1)))  # [c, n*q, a]
        F = F.reshape(nc, n, nq * 3)
        if det is not None:
            F /= det[:, None, None]
        return F @ np.transpose(F, (0, 2, 1))

    def element_matrices(self, cells, alpha, beta):
        """[nc, n, n] element matrices of a^k on the given cells, by quadrature
        of the physical basis functions (R-A10): the pulled-back values at the
        quadrature points (J^-T grad for 0-forms, J^-T phi / J curl / det for
        1-forms, J phi / det and div / det for 2-forms), weighted sums over points."""
        J = self.jacobians(cells)
        det = np.linalg.det(J)
        vol = np.abs(det) * self.vol_hat
        if self.space == "hgrad":
            Jit = np.linalg.inv(np.transpose(J, (0, 2, 1)))   # J^-T
            Vw = self._weighted("val")                       # [n, q]
            Mm = Vw @ Vw.T
            Kk = self._gram_phys(Jit, self._weighted("der"))  # physical gradients
            return vol[:, None, None] * (beta[:, None, None] * Mm[None] + alpha[:, None, None] * Kk)
        if self.space == "hdiv":  # 2-forms: phi = J phi-hat / det J, div phi = div-hat phi-hat / det J
            Mm = self._gram_phys(J, self._weighted("val"), det)
            Dw = self._weighted("der")[None] / det[:, None, None]  # [c, n, q]
            Kk = Dw @ np.transpose(Dw, (0, 2, 1))
            return vol[:, None, None] * (beta[:, None, None] * Mm + alpha[:, None, None] * Kk)
        Jit = np.linalg.inv(np.transpose(J, (0, 2, 1)))
        Mm = self._gram_phys(Jit, self._weighted("val"))
        Kk = self._gram_phys(J, self._weighted("der"), det)
        return vol[:, None, None] * (beta[:, None, None] * Mm + alpha[:, None, None] * Kk)

    def assemble(self, alpha, beta, chunk: int = 256):
        """Global CSR of a^k over all dofs (constrained rows/cols included)."""
        nt, n = self.topo.nt, self.el.n
        N = self.num.n_total
        mats = []
        for c0 in range(0, nt, chunk):
            cells = np.arange(c0, min(nt, c0 + chunk))
            Ae = self.element_matrices(cells, alpha[cells], beta[cells])
            dm = self.num.dofmap[cells]
            rows = np.repeat(dm, n, axis=1).ravel()
            cols = np.tile(dm, (1, n)).ravel()
            mats.append(sp.csr_matrix((Ae.ravel(), (rows, cols)), shape=(N, N)))
        A = mats[0]
        for m in mats[1:]:
            A = A + m
        A.sum_duplicates()
        return A.tocsr()
