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

    def element_matrices(self, cells, alpha, beta):
        """[nc, n, n] element matrices of a^k on the given cells."""
        J = self.jacobians(cells)
        det = np.linalg.det(J)
        vol = np.abs(det) * self.vol_hat
        wq = self.w
        sw = np.sqrt(wq)

        def gram(F):  # sum_q w_q F[c,q,i,:].F[c,q,j,:] as a batched matmul
            G = np.transpose(F * sw[None, :, None, None], (0, 2, 1, 3)).reshape(F.shape[0], F.shape[2], -1)
            return G @ np.transpose(G, (0, 2, 1))

        if self.space == "hgrad":
            Jit = np.linalg.inv(np.transpose(J, (0, 2, 1)))   # J^-T
            g = np.einsum("cab,qnb->cqna", Jit, self.der)     # physical gradients
            Mm = np.einsum("q,qi,qj->ij", wq, self.val, self.val)
            Kk = gram(g)
            return vol[:, None, None] * (beta[:, None, None] * Mm[None] + alpha[:, None, None] * Kk)
        if self.space == "hdiv":  # 2-forms: phi = J phi-hat / det J, div phi = div-hat phi-hat / det J
            ph = np.einsum("cab,qnb->cqna", J, self.val) / det[:, None, None, None]
            dv = self.der[None] / det[:, None, None]
            Mm = gram(ph)
            Kk = np.einsum("q,cqi,cqj->cij", wq, dv, dv)
            return vol[:, None, None] * (beta[:, None, None] * Mm + alpha[:, None, None] * Kk)
        Jit = np.linalg.inv(np.transpose(J, (0, 2, 1)))
        ph = np.einsum("cab,qnb->cqna", Jit, self.val)
        cu = np.einsum("cab,qnb->cqna", J, self.der) / det[:, None, None, None]
        Mm = gram(ph)
        Kk = gram(cu)
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
