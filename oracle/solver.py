"""Operator, one-level additive preconditioner and PCG of the hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Preconditioner (DESIGN.md R-A13..A15, R-A17):
  P^-1 r = sum_{l in I} e_l r_l / A_ll + sum_m E_m (E_m^T A E_m)^-1 E_m^T r
  * interior point-Jacobi on all cell-interior dofs (Thm 5.1)
  * H(grad): one patch per vertex V = free interface dofs of V, the edges
    and the faces containing V: PAFW0(X0_Gamma) + J(X0_I) (Eq. 5.4)
  * H(curl): PH(X0_Gamma, X^{1,I}_Gamma) + J(X1_I) (Eq. 5.12):
    vertex potential patches E_m = G_V (discrete gradient columns of the free
    CG_p interface dofs of the vertex star) and edge patches = free Whitney dof
    of E + type-I dofs of the faces containing E.
  * H(div): PAFW1(X2_Gamma) + J(X2_I) (Eq. 5.16):
    one patch per edge E = the free dofs of the faces containing E.
  Local solvers are exact: dense Cholesky (scipy cho_factor/cho_solve).
PCG (R-A16): x0 = 0, stop when ||z||_2 <= rtol ||z0||_2 (P:2326-2328 gives rtol 1e-8).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.linalg as sla

from .mesh import Topology, number, dofs_per_entity, dof_layout
from .refelem import element
from .fem import Assembler


class Oracle:
    def __init__(self, vertices, tets, p, space, alpha, beta, mask, assemble=True, decomposition="split"):
        self.space = {0: "hgrad", 1: "hcurl", 2: "hdiv", "hgrad": "hgrad", "hcurl": "hcurl", "hdiv": "hdiv"}[space]
        self.p = p
        # "split": PAFW0(X_Gamma)+J(X_I) (Eq. 5.4) / PH(X0_Gamma, X1I_Gamma)+J(X1_I) (Eq. 5.12), the hot path;
        # "unsplit": PAFW0(X) (Eq. 5.2) / PH(X0, X1I) (Eq. 5.10), interiors inside the star patches and
        # no Jacobi; both one-level (the coarse W^k is NEXT-1, R-A14)
        assert decomposition in ("split", "unsplit")
        self.decomposition = decomposition
        self.alpha = np.asarray(alpha, dtype=np.float64)
        self.beta = np.asarray(beta, dtype=np.float64)
        self.topo = Topology(vertices, tets, mask)
        self.num = number(self.space, p, self.topo, dof_layout(self.space, p))
        self.n_total = self.num.n_total
        self.free = ~self.num.constrained
        self.A = None
        self._patches = None
        self._asm = None
        if assemble:
            self.assemble()

    @property
    def el(self):
        return element(self.space, self.p)

    @property
    def asm(self):
        if self._asm is None:
            self._asm = Assembler(self.space, self.p, self.topo, self.num)
        return self._asm

    # ------------------------------------------------------------ operator
    def assemble(self):
        A = self.asm.assemble(self.alpha, self.beta)
        f = self.free.astype(np.float64)
        Dg = sp.diags(f)
        self.A = (Dg @ A @ Dg).tocsr()     # A_FF embedded, constrained rows/cols zero
        self.A.eliminate_zeros()
        return self.A

    def mask(self, x):
        x = np.array(x, dtype=np.float64, copy=True)
        x[~self.free] = 0.0
        return x

    def apply(self, x):
        """y = A x with y_F = A_FF x_F, y_D = 0 (Eq. 2.9 / R-A11)."""
        return self.A @ self.mask(x)

    # ------------------------------------------------------------ patches
    def _incidence(self):
        """vertex -> incident edges / faces, edge -> incident faces (cached)."""
        if getattr(self, "_inc", None) is None:
            t = self.topo
            v_edges = [[] for _ in range(t.nv)]
            for e, (a, b) in enumerate(t.edges):
                v_edges[a].append(e)
                v_edges[b].append(e)
            v_faces = [[] for _ in range(t.nv)]
            for f, tri in enumerate(t.faces):
                for a in tri:
                    v_faces[a].append(f)
            e_faces = [[] for _ in range(t.ne)]
            for f, tri in enumerate(t.faces):
                for a, b in ((0, 1), (0, 2), (1, 2)):
                    e_faces[t.edge_index[(tri[a], tri[b])]].append(f)
            self._inc = (v_edges, v_faces, e_faces)
        return self._inc

    def _cells_of(self, verts):
        """Cells containing all of the given vertices (the star of a vertex / edge)."""
        return np.nonzero(np.sum(np.isin(self.topo.cells, verts), axis=1) == len(verts))[0]

    def vertex_patch(self, v):
        """(kind, idx) of the star patch of vertex v (R-A13): the free interface
        dofs of v, the edges and the faces containing v -- in the problem's own
        numbering for H(grad) ('dof'), in the CG_p potential numbering for
        H(curl) ('pot', embedded by G[:, idx]). Unsplit (Eq. 5.2 / 5.10): also
        the interior dofs of the cells containing v. Empty idx: no patch."""
        v_edges, v_faces, _ = self._incidence()
        num = self.num if self.space == "hgrad" else (self._build_gradient(), self.cg_num)[1]
        idx = self._entity_dofs(num, v, v_edges[v], v_faces[v], kinds=None)
        if self.decomposition == "unsplit" and num.per[3]:
            cells = self._cells_of([v])
            o, per = num.offsets[3], num.per[3]
            idx = np.sort(np.concatenate([idx] + [np.arange(o + c * per, o + (c + 1) * per) for c in cells]))
        if self.space == "hgrad":
            return "dof", idx[self.free[idx]]
        return "pot", idx[~num.constrained[idx]]

    def edge_patch(self, e):
        """('dof', idx) of the type-I edge patch of E (H(curl), R-A13): the free
        Whitney dof of E and the type-I dofs of the faces containing E; unsplit
        (Eq. 5.10) also the type-I dofs of the cells containing E.
        H(div) (Eq. 5.16, DESIGN.md R-D3): X^2_Gamma restricted to
        the edge star = every free dof of the faces containing E; unsplit
        (PAFW1(X^2)) also every dof of the cells containing E."""
        _, _, e_faces = self._incidence()
        num = self.num
        if self.space == "hdiv":
            idx = []
            for f in e_faces[e]:
                base = num.offsets[2] + f * num.per[2]
                idx.extend(range(base, base + num.per[2]))
            if self.decomposition == "unsplit":
                for c in self._cells_of(list(self.topo.edges[e])):
                    base = num.offsets[3] + c * num.per[3]
                    idx.extend(range(base, base + num.per[3]))
            idx = np.array(sorted(idx), dtype=np.int64)
            return "dof", idx[self.free[idx]]
        nI_face = num.per[2] - (self.p - 1) * (self.p - 2) // 2
        idx = [num.offsets[1] + e * num.per[1]]       # Whitney dof of E
        for f in e_faces[e]:
            base = num.offsets[2] + f * num.per[2]
            idx.extend(range(base, base + nI_face))  # type-I face dofs
        if self.decomposition == "unsplit":
            nI_cell = num.per[3] - (self.p - 1) * (self.p - 2) * (self.p - 3) // 6
            for c in self._cells_of(list(self.topo.edges[e])):
                base = num.offsets[3] + c * num.per[3]
                idx.extend(range(base, base + nI_cell))  # type-I cell dofs
        idx = np.array(sorted(idx), dtype=np.int64)
        return "dof", idx[self.free[idx]]

    def patch_sets(self):
        """List of (kind, idx) with idx global dof ids; for kind 'pot' idx are
        CG_p dof ids of the potential space and the embedding is G[:, idx]."""
        if self._patches is not None:
            return self._patches
        out = []
        for v in range(self.topo.nv if self.space != "hdiv" else 0):  # H(div): edge stars only (Eq. 5.16)
            kind, idx = self.vertex_patch(v)
            if len(idx):
                out.append((kind, idx))
        if self.space in ("hcurl", "hdiv"):
            for e in range(self.topo.ne):
                kind, idx = self.edge_patch(e)
                if len(idx):
                    out.append((kind, idx))
        self._patches = out
        return out

    @staticmethod
    def _entity_dofs(num, v, edges, faces, kinds):
        ids = []
        o, per = num.offsets, num.per
        if per[0]:
            ids.append(o[0] + v)
        for e in edges:
            ids.extend(range(o[1] + e * per[1], o[1] + (e + 1) * per[1]))
        for f in faces:
            ids.extend(range(o[2] + f * per[2], o[2] + (f + 1) * per[2]))
        return np.array(sorted(ids), dtype=np.int64)

    def _build_gradient(self):
        """Discrete gradient G: CG_p dofs -> Ned1_p dofs (R-A12, Lemma 4.1 + 4.3):
        G[Whitney(E), V] = +1 if V is the higher vertex of E, -1 if the lower;
        G[typeII(S,j), CGbubble(S,j)] = +1 for S = edge, face, cell."""
        if hasattr(self, "G"):
            return self.G
        self.cg_num = number("hgrad", self.p, self.topo, dof_layout("hgrad", self.p))
        cg, ned, t, p = self.cg_num, self.num, self.topo, self.p
        rows, cols, vals = [], [], []
        for e, (a, b) in enumerate(t.edges):
            w = ned.offsets[1] + e * ned.per[1]
            rows += [w, w]
            cols += [a, b]
            vals += [-1.0, 1.0]
            for j in range(p - 1):
                rows.append(w + 1 + j)
                cols.append(cg.offsets[1] + e * cg.per[1] + j)
                vals.append(1.0)
        nI_face = ned.per[2] - cg.per[2]
        for f in range(t.nf):
            for j in range(cg.per[2]):
                rows.append(ned.offsets[2] + f * ned.per[2] + nI_face + j)
                cols.append(cg.offsets[2] + f * cg.per[2] + j)
                vals.append(1.0)
        nI_cell = ned.per[3] - cg.per[3]
        for c in range(t.nt):
            for j in range(cg.per[3]):
                rows.append(ned.offsets[3] + c * ned.per[3] + nI_cell + j)
                cols.append(cg.offsets[3] + c * cg.per[3] + j)
                vals.append(1.0)
        self.G = sp.csr_matrix((vals, (rows, cols)), shape=(ned.n_total, cg.n_total))
        return self.G

    def _potential_operator(self):
        """(grad phi_i, beta grad phi_j) on CG_p (Eq. 5.11), free CG dofs only."""
        if getattr(self, "_Apot", None) is None:
            self._build_gradient()
            asm = Assembler("hgrad", self.p, self.topo, self.cg_num)
            K = asm.assemble(self.beta, np.zeros_like(self.beta))
            f = sp.diags((~self.cg_num.constrained).astype(np.float64))
            self._Apot = (f @ K @ f).tocsr()
        return self._Apot

    def build_preconditioner(self, kappa: bool = True):
        """Factor every patch matrix; kappa=True also records max kappa(A_m)
        (the oracle reports it next to the 1e-11 parity bar)."""
        Ar = self.A
        d = Ar.diagonal()
        # interior point-Jacobi only in the split decompositions (Thm 5.1); unsplit
        # patches contain the interiors
        self.int_idx = np.nonzero(self.num.interior & self.free)[0] if self.decomposition == "split" \
            else np.zeros(0, dtype=np.int64)
        self.dinv = 1.0 / d[self.int_idx]
        self.factors = []
        self.kappa_max = 0.0
        for kind, idx in self.patch_sets():
            if kind == "dof":
                Am = Ar[idx][:, idx].toarray()
                emb = None
            else:
                # Eq. 5.11: the local potential problem is
                # (d phi, beta d psi) on the star, i.e. the beta-weighted CG_p
                # stiffness (= G_V^T A G_V since curl grad = 0, pinned in
                # test_hcurl_gradients), assembled by physical quadrature.
                Gv = self.G[:, idx]
                Am = self._potential_operator()[idx][:, idx].toarray()
                emb = Gv.tocsr()
            if kappa:
                ev = np.linalg.eigvalsh(Am)
                if ev[0] <= 0:
                    raise np.linalg.LinAlgError("patch matrix not SPD")
                self.kappa_max = max(self.kappa_max, ev[-1] / ev[0])
            self.factors.append((kind, idx, emb, sla.cho_factor(Am, lower=True)))
        return self

    def precond(self, r):
        """z = P^-1 r (one-level additive, R-A14)."""
        if not hasattr(self, "factors"):
            self.build_preconditioner()
        r = self.mask(r)
        z = np.zeros_like(r)
        z[self.int_idx] += self.dinv * r[self.int_idx]
        for kind, idx, emb, fac in self.factors:
            if kind == "dof":
                z[idx] += sla.cho_solve(fac, r[idx])
            else:
                u = sla.cho_solve(fac, emb.T @ r)
                z += emb @ u
        z[~self.free] = 0.0
        return z

    # ------------------------------------------------------------ PCG
    def solve(self, b, rtol=1e-8, maxit=10000, history=None):
        """PCG per R-A16. Returns (x, iters, true relative residual); `history`
        (a list) receives ||z_k|| / ||z_0|| for k = 1..iters."""
        b = self.mask(b)
        x = np.zeros_like(b)
        r = b.copy()
        z = self.precond(r)
        z0 = np.linalg.norm(z)
        if z0 == 0:
            return x, 0, 0.0
        pv = z.copy()
        rho = r @ z
        it = 0
        for k in range(maxit):
            q = self.apply(pv)
            a = rho / (pv @ q)
            x += a * pv
            r -= a * q
            z = self.precond(r)
            it = k + 1
            if history is not None:
                history.append(np.linalg.norm(z) / z0)
            if np.linalg.norm(z) <= rtol * z0:
                break
            rho_new = r @ z
            pv = z + (rho_new / rho) * pv
            rho = rho_new
        res = np.linalg.norm(b - self.apply(x)) / np.linalg.norm(b)
        return x, it, res
