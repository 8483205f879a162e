"""Sampled rows of A x and P^-1 r for meshes too large to assemble globally.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY §8(c) "Config 3 oracle scope": at full size the global CSR of the
oracle does not fit the parity budget, so the operator and the preconditioner
are checked on sampled output rows that the oracle computes one by one from
the same definitions as oracle.solver.Oracle:

  * (A x)_r = sum over cells T containing dof r of (A_T x_T)_r, with A_T the
    element matrix by physical quadrature (Eq. 2.9, R-A10) and x
    masked (R-A11); y_r = 0 for constrained r.
  * (P^-1 r)_l = r_l / A_ll for interior l (split decompositions: Thm 5.1,
    P:1612-1631, R-A17), plus
    sum over the star patches m containing l of (E_m A_m^-1 E_m^T r)_l
    (Eq. 5.4; Eq. 5.12, R-A13..A15). A_m is assembled
    from the element matrices of the cells of the star only -- every cell that
    couples two dofs of the patch contains the seed vertex (edge), so this is
    exactly A[idx][:, idx]. The patches that can contain a dof of an entity S
    are the vertex patches of the vertices of S and (H(curl)) the edge patches
    of the edges of S; the others contribute 0 at that row. (The unsplit
    decompositions of SURVEY NEXT-3 put interior dofs into the patches too.)
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .fem import Assembler
from .solver import Oracle


class SampledOracle(Oracle):
    def __init__(self, vertices, tets, p, space, alpha, beta, mask, decomposition="split"):
        super().__init__(vertices, tets, p, space, alpha, beta, mask, assemble=False, decomposition=decomposition)
        self._Ae = {}
        self._Ae_cg = {}
        self._solved = {}

    # ------------------------------------------------------------ element matrices
    def _elements(self, cells, potential=False):
        """{cell: element matrix}; own space, or the beta-weighted CG_p
        stiffness of the H(curl) potential patches (Eq. 5.11)."""
        cache = self._Ae_cg if potential else self._Ae
        missing = np.array(sorted(set(int(c) for c in cells) - set(cache)), dtype=np.int64)
        if len(missing):
            if potential:
                self._build_gradient()
                if getattr(self, "_asm_cg", None) is None:
                    self._asm_cg = Assembler("hgrad", self.p, self.topo, self.cg_num)
                mats = self._asm_cg.element_matrices(missing, self.beta[missing], np.zeros(len(missing)))
            else:
                mats = self.asm.element_matrices(missing, self.alpha[missing], self.beta[missing])
            for c, m in zip(missing, mats):
                cache[int(c)] = m
        return {int(c): cache[int(c)] for c in cells}

    # ------------------------------------------------------------ operator rows
    def apply_rows(self, x, rows):
        """(A_FF x_F)_r for r in rows (0 for constrained r)."""
        xm = self.mask(x)
        rows = np.asarray(rows, dtype=np.int64)
        dm = self.num.dofmap
        hit = np.isin(dm, rows)
        cells = np.nonzero(hit.any(axis=1))[0]
        Ae = self._elements(cells)
        out = {int(r): 0.0 for r in rows}
        for c in cells:
            loc = np.nonzero(hit[c])[0]
            yc = Ae[int(c)][loc] @ xm[dm[c]]
            for k, yv in zip(loc, yc):
                out[int(dm[c, k])] += yv
        y = np.array([out[int(r)] for r in rows])
        y[~self.free[rows]] = 0.0
        return y

    # ------------------------------------------------------------ preconditioner rows
    def _patch_solve(self, kind, seed, r):
        """Correction of one patch in the problem's numbering, as (dof ids,
        values); memoised per (kind, seed) for the current r."""
        key = (kind, seed)
        if key in self._solved:
            return self._solved[key]
        if kind == "vertex":
            pk, idx = self.vertex_patch(seed)
            cells = self._cells_of([seed])
        else:
            pk, idx = self.edge_patch(seed)
            cells = self._cells_of(list(self.topo.edges[seed]))
        if len(idx) == 0:
            self._solved[key] = (np.zeros(0, dtype=np.int64), np.zeros(0))
            return self._solved[key]
        pot = pk == "pot"
        num = self.cg_num if pot else self.num
        Ae = self._elements(cells, potential=pot)
        pos = {int(g): i for i, g in enumerate(idx)}
        n = len(idx)
        Am = np.zeros((n, n))
        for c in cells:
            g = num.dofmap[c]
            loc = [k for k in range(len(g)) if int(g[k]) in pos]
            pl = [pos[int(g[k])] for k in loc]
            Am[np.ix_(pl, pl)] += Ae[int(c)][np.ix_(loc, loc)]
        fac = sla.cho_factor(Am, lower=True)
        if pot:
            Gv = self.G[:, idx].tocsc()
            u = sla.cho_solve(fac, Gv.T @ r)
            corr = Gv @ u
            ids = np.nonzero(corr)[0]
            res = (ids, corr[ids])
        else:
            res = (idx, sla.cho_solve(fac, r[idx]))
        self._solved[key] = res
        return res

    def _candidate_seeds(self, l):
        """Patches (kind, seed) that can contain dof l: the vertex patches of the
        vertices of its entity and (H(curl)) the edge patches of its edges."""
        t = self.topo
        dim, ent = self.num.entity[l]
        verts = [int(ent)] if dim == 0 else list(t.edges[ent]) if dim == 1 else \
            list(t.faces[ent]) if dim == 2 else list(t.cells[ent])
        if self.space == "hdiv":  # edge stars only: the edges of the dof's face (cell, unsplit)
            vs = sorted(verts)
            return [("edge", t.edge_index[(vs[ia], vs[ib])]) for ia in range(len(vs)) for ib in range(ia + 1, len(vs))]
        seeds = [("vertex", v) for v in verts]
        if self.space == "hcurl" and dim >= 1:
            vs = sorted(verts)
            for ia in range(len(vs)):
                for ib in range(ia + 1, len(vs)):
                    seeds.append(("edge", t.edge_index[(vs[ia], vs[ib])]))
        return seeds

    def precond_residual_rows(self, b, x, rows):
        """(P^-1 (b - A x))_l for l in rows, with the residual formed by the
        oracle on every dof the relevant patches touch (the other entries of r
        do not enter these rows) -- the quantity of the PCG stopping rule R-A16
        at a solution x, on sampled rows."""
        rows = np.asarray(rows, dtype=np.int64)
        need = set(int(l) for l in rows)
        for l in rows:
            if not self.free[l]:
                continue
            if self.num.entity[l][0] == 3 and self.decomposition == "split":
                continue
            for kind, seed in self._candidate_seeds(int(l)):
                pk, idx = self.vertex_patch(seed) if kind == "vertex" else self.edge_patch(seed)
                if pk == "pot":  # Ned1 dofs reached by G_V^T
                    idx = np.nonzero(np.abs(self.G[:, idx]).sum(axis=1).A1)[0]
                need.update(int(i) for i in idx)
        need = np.array(sorted(need), dtype=np.int64)
        r = np.zeros(self.n_total)
        r[need] = self.mask(b)[need] - self.apply_rows(x, need)
        return self.precond_rows(r, rows)

    def precond_rows(self, r, rows):
        """(P^-1 r)_l for l in rows (0 for constrained l)."""
        r = self.mask(r)
        self._solved = {}
        rows = np.asarray(rows, dtype=np.int64)
        out = np.zeros(len(rows))
        for i, l in enumerate(rows):
            if not self.free[l]:
                continue
            dim, ent = self.num.entity[l]
            if dim == 3 and self.decomposition == "split":  # interior point-Jacobi, d_l = A_ll (R-A17)
                c = int(ent)
                k = int(np.nonzero(self.num.dofmap[c] == l)[0][0])
                out[i] += r[l] / self._elements([c])[c][k, k]
                continue
            for kind, seed in self._candidate_seeds(int(l)):
                ids, vals = self._patch_solve(kind, seed, r)
                hit = np.nonzero(ids == l)[0]
                if len(hit):
                    out[i] += vals[hit[0]]
        return out
