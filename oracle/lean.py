"""Memory-lean oracle: the same operator, preconditioner and PCG as
oracle.solver.Oracle, for meshes whose global CSR does not fit the host.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY §8(c) "Config 3 oracle scope": the global CSR of config 3 has
nnz ~ 1.7e9 and its COO build ~ 2e9 triplets, more than this oracle's hosts
hold alongside the patch factors. This class computes exactly what
Oracle computes, from the same definitions, with less memory:

  * A x = sum_T E_T A_T E_T^T x (the element-by-element form of the same
    assembly, Eq. 2.9), with A_T the element matrix by physical
    quadrature (oracle.fem.Assembler.element_matrices, R-A10) kept per cell
    (optionally in a disk-backed array); x masked and y_D = 0 (R-A11).
  * d_l = A_ll for interior l (R-A17): an interior dof belongs to one cell,
    so this is that cell's element diagonal (Thm 5.1).
  * A_m = E_m^T A E_m assembled from the element matrices of the cells of the
    star only (every cell coupling two dofs of a star contains its seed
    vertex / edge -- the argument of oracle/sampled.py), potential patches of
    H(curl) from the beta-weighted CG_p stiffness (Eq. 5.11) and
    embedded by G_V (Eq. 5.12); exact local solves (R-A15) by a Cholesky
    factorisation in LAPACK's packed storage (dpptrf / dpptrs), so that each
    factor takes n(n+1)/2 doubles instead of n^2.
  * PCG: Oracle.solve unchanged (R-A16).

Pinned against Oracle (vector by vector and iteration counts) on small meshes
of all three spaces in tests/test_oracle_lean.py.
"""
from __future__ import annotations

import os
import tempfile

import numpy as np
from scipy.linalg import lapack

from .fem import Assembler
from .solver import Oracle


_WORK = None


def _single_thread():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _run_work(c0):
    return _WORK(c0)


class LeanOracle(Oracle):
    def __init__(self, vertices, tets, p, space, alpha, beta, mask, store_dir: str | None = None,
                 chunk: int = 64, verbose: bool = False, workers: int = 1):
        super().__init__(vertices, tets, p, space, alpha, beta, mask, assemble=False)
        self.store_dir = store_dir
        self.chunk = chunk
        self.workers = workers if store_dir is not None else 1  # workers share a disk-backed array
        self.verbose = verbose
        self.Ae = self._element_store(self.asm, self.alpha, self.beta, "Ae")

    def _log(self, msg):
        if self.verbose:
            print(f"[lean] {msg}", flush=True)

    def _array(self, name, shape):
        if self.store_dir is None:
            return np.empty(shape, dtype=np.float64)
        fd, path = tempfile.mkstemp(prefix=f"lean_{name}_", suffix=".npy", dir=self.store_dir)
        os.close(fd)
        arr = np.lib.format.open_memmap(path, mode="w+", dtype=np.float64, shape=shape)
        os.unlink(path)  # the mapping keeps the file alive until the array is dropped
        return arr

    def _element_store(self, asm, alpha, beta, name):
        nt, n = self.topo.nt, asm.el.n
        Ae = self._array(name, (nt, n, n))
        starts = list(range(0, nt, self.chunk))

        def work(c0):
            cells = np.arange(c0, min(nt, c0 + self.chunk))
            Ae[cells] = asm.element_matrices(cells, alpha[cells], beta[cells])
            return c0

        if self.workers <= 1:
            for c0 in starts:
                work(c0)
                if c0 % (self.chunk * 64) == 0:
                    self._log(f"{name}: {c0}/{nt} cells")
        else:  # forked workers write disjoint cells of the shared (MAP_SHARED) array
            import multiprocessing as mp
            global _WORK
            _WORK = work
            with mp.get_context("fork").Pool(self.workers, initializer=_single_thread) as pool:
                for i, _ in enumerate(pool.imap_unordered(_run_work, starts)):
                    if i % 64 == 0:
                        self._log(f"{name}: {i * self.chunk}/{nt} cells")
            Ae.flush()
        return Ae

    # ------------------------------------------------------------ operator
    def apply(self, x):
        """y = A x with y_F = A_FF x_F, y_D = 0 (Eq. 2.9 / R-A11)."""
        xm = self.mask(x)
        dm = self.num.dofmap
        y = np.zeros(self.n_total)
        for c0 in range(0, self.topo.nt, 1024):
            sl = slice(c0, min(self.topo.nt, c0 + 1024))
            Y = np.matmul(self.Ae[sl], xm[dm[sl]][:, :, None])[:, :, 0]
            y += np.bincount(dm[sl].ravel(), weights=Y.ravel(), minlength=self.n_total)
        y[~self.free] = 0.0
        return y

    # ------------------------------------------------------------ preconditioner
    def _star_cells(self):
        """vertex -> cells containing it (the stars of A13)."""
        if getattr(self, "_vcells", None) is None:
            cells = self.topo.cells
            order = np.argsort(cells.ravel(), kind="stable")
            counts = np.bincount(cells.ravel(), minlength=self.topo.nv)
            ptr = np.concatenate([[0], np.cumsum(counts)])
            self._vcells = (ptr, order // 4)
        return self._vcells

    def _cells_of(self, verts):
        ptr, cl = self._star_cells()
        s = set(cl[ptr[verts[0]]:ptr[verts[0] + 1]].tolist())
        for v in verts[1:]:
            s &= set(cl[ptr[v]:ptr[v + 1]].tolist())
        return np.array(sorted(s), dtype=np.int64)

    def _patch_matrix(self, cells, idx, num, Ae):
        pos = np.full(num.n_total, -1, dtype=np.int64)
        pos[idx] = np.arange(len(idx))
        n = len(idx)
        Am = np.zeros((n, n))
        for c in cells:
            pl = pos[num.dofmap[c]]
            loc = np.nonzero(pl >= 0)[0]
            pl = pl[loc]
            Am[np.ix_(pl, pl)] += Ae[c][np.ix_(loc, loc)]
        return Am

    def build_preconditioner(self, kappa: bool = False):
        """Interior point-Jacobi (split, R-A17) and one packed Cholesky factor per
        star patch (R-A13..A15), in the order of Oracle.patch_sets()."""
        assert self.decomposition == "split"
        nt = self.topo.nt
        self.int_idx = np.nonzero(self.num.interior & self.free)[0]
        diag = np.zeros(self.n_total)
        for c0 in range(0, nt, 1024):
            sl = slice(c0, min(nt, c0 + 1024))
            dm = self.num.dofmap[sl]
            d = np.diagonal(self.Ae[sl], axis1=1, axis2=2)
            inter = self.num.interior[dm]
            diag[dm[inter]] = d[inter]          # one cell per interior dof: no sum
        self.dinv = 1.0 / diag[self.int_idx]
        Ae_pot = None
        if self.space == "hcurl":
            self._build_gradient()
            asm_cg = Assembler("hgrad", self.p, self.topo, self.cg_num)
            Ae_pot = self._element_store(asm_cg, self.beta, np.zeros_like(self.beta), "Ae_pot")
        sets = self.patch_sets()
        sizes = np.array([len(idx) for _, idx in sets], dtype=np.int64)
        offs = np.concatenate([[0], np.cumsum(sizes * (sizes + 1) // 2)])
        self.packed = self._array("factors", (int(offs[-1]),))
        self.factors = []
        nv = self.topo.nv if self.space != "hdiv" else 0
        k = 0
        if nv:  # vertex patches (patch_sets order: vertices ascending, nonempty only)
            for v in range(nv):
                kind, idx = self.vertex_patch(v)
                if not len(idx):
                    continue
                assert np.array_equal(idx, sets[k][1])
                cells = self._cells_of([v])
                if kind == "dof":
                    Am = self._patch_matrix(cells, idx, self.num, self.Ae)
                    emb = None
                else:
                    Am = self._patch_matrix(cells, idx, self.cg_num, Ae_pot)
                    emb = self.G[:, idx].tocsr()
                self._factor(k, Am, offs, kind, idx, emb)
                k += 1
                if k % 512 == 0:
                    self._log(f"patches: {k}/{len(sets)}")
        if self.space in ("hcurl", "hdiv"):
            for e in range(self.topo.ne):
                kind, idx = self.edge_patch(e)
                if not len(idx):
                    continue
                assert np.array_equal(idx, sets[k][1])
                cells = self._cells_of(list(self.topo.edges[e]))
                Am = self._patch_matrix(cells, idx, self.num, self.Ae)
                self._factor(k, Am, offs, kind, idx, None)
                k += 1
        assert k == len(sets)
        del Ae_pot
        return self

    def _factor(self, k, Am, offs, kind, idx, emb):
        n = Am.shape[0]
        ap = Am[np.triu_indices(n)]             # column-major lower packed == row-major upper (symmetric)
        ap, info = lapack.dpptrf(n, ap, lower=1)
        if info != 0:
            raise np.linalg.LinAlgError("patch matrix not SPD")
        self.packed[offs[k]:offs[k + 1]] = ap
        self.factors.append((kind, idx, emb, (int(offs[k]), int(offs[k + 1]), n)))

    def precond(self, r):
        """z = P^-1 r (one-level additive, R-A14)."""
        if not hasattr(self, "factors"):
            self.build_preconditioner()
        r = self.mask(r)
        z = np.zeros_like(r)
        z[self.int_idx] += self.dinv * r[self.int_idx]
        for kind, idx, emb, (o0, o1, n) in self.factors:
            rhs = r[idx] if kind == "dof" else emb.T @ r
            u, info = lapack.dpptrs(n, self.packed[o0:o1], rhs[:, None], lower=1)
            assert info == 0
            u = u[:, 0]
            if kind == "dof":
                z[idx] += u
            else:
                z += emb @ u
        z[~self.free] = 0.0
        return z


class IterationSample:
    """A bounded sample of one LeanOracle PCG iteration on a full-size workload
    (bench.py's cpu_baseline and --impl reference legs, SURVEY §8(d) "Oracle
    timing beside it"). Per iteration LeanOracle does one element-by-element
    apply over every cell, one packed Cholesky solve per star patch (plus the
    interior Jacobi) and O(N) vector work. The sample: the n_patches vertex
    patches nearest the centre of the mesh and the cells of their stars
    (setup of both untimed, as for the full oracle). time_iteration() times the
    sample's apply and patch solves and the full-length vector work, and scales
    the first two to the whole mesh by cells and by packed-factor doubles:
        t_iter = t_apply(sample) * n_cells / n_cells(sample)
               + t_patches(sample) * sum_m n_m(n_m+1)/2 / sum_sample n_m(n_m+1)/2
               + t_vector(full length)."""

    def __init__(self, O: Oracle, n_patches: int = 32, workers: int = 1):
        self.O = O
        t = O.topo
        assert O.space == "hgrad", "the sample covers the H(grad) vertex stars"
        centre = t.vertices.mean(axis=0)
        order = np.argsort(np.linalg.norm(t.vertices - centre, axis=1), kind="stable")
        self.patches = []
        lean = LeanOracle.__new__(LeanOracle)  # helpers only (star cells, patch assembly, packed factor)
        lean.__dict__.update(O.__dict__)
        lean.verbose = False
        for v in order:
            kind, idx = O.vertex_patch(int(v))
            if len(idx) and not t.dir_vertex[v]:
                self.patches.append((int(v), idx))
            if len(self.patches) == n_patches:
                break
        cells = np.unique(np.concatenate([lean._cells_of([v]) for v, _ in self.patches]))
        self.cells = cells
        Ae = np.empty((len(cells), O.asm.el.n, O.asm.el.n))
        for c0 in range(0, len(cells), 64):
            cc = cells[c0:c0 + 64]
            Ae[c0:c0 + len(cc)] = O.asm.element_matrices(cc, O.alpha[cc], O.beta[cc])
        self.Ae = Ae
        pos = {int(c): i for i, c in enumerate(cells)}
        self.factors = []
        for v, idx in self.patches:
            sc = lean._cells_of([v])
            Am = lean._patch_matrix([pos[int(c)] for c in sc], idx, _Renumbered(O.num, sc, cells), Ae)
            n = len(idx)
            ap, info = lapack.dpptrf(n, Am[np.triu_indices(n)], lower=1)
            assert info == 0
            self.factors.append((idx, ap, n))
        sizes = np.array([len(idx) for _, idx in O.patch_sets()], dtype=np.float64)
        self.scale_apply = t.nt / len(cells)
        self.scale_patches = float(np.sum(sizes * (sizes + 1) / 2)) / float(
            sum(n * (n + 1) / 2 for _, _, n in self.factors))
        self.int_idx = np.nonzero(O.num.interior & O.free)[0]

    def time_iteration(self, rng_seed: int = 0):
        import time
        O = self.O
        rng = np.random.default_rng(rng_seed)
        x = O.mask(rng.uniform(-1, 1, O.n_total))
        dm = O.num.dofmap[self.cells]
        t0 = time.perf_counter()
        Y = np.matmul(self.Ae, x[dm][:, :, None])[:, :, 0]
        y = np.bincount(dm.ravel(), weights=Y.ravel(), minlength=O.n_total)
        y[~O.free] = 0.0
        t1 = time.perf_counter()
        z = np.zeros(O.n_total)
        for idx, ap, n in self.factors:
            u, info = lapack.dpptrs(n, ap, x[idx][:, None], lower=1)
            z[idx] += u[:, 0]
        t2 = time.perf_counter()
        # the full-length vector work of Oracle.solve's loop body (+ interior Jacobi)
        r, pv, q, xs = x.copy(), x.copy(), y, np.zeros(O.n_total)
        a = (r @ x) / (pv @ q + 1.0)
        xs += a * pv
        r -= a * q
        zz = np.zeros_like(r)
        zz[self.int_idx] += r[self.int_idx]
        zz[~O.free] = 0.0
        nz = np.linalg.norm(zz)
        rho = r @ zz
        pv = zz + (rho / (nz + 1.0)) * pv
        t3 = time.perf_counter()
        t_apply, t_patch, t_vec = t1 - t0, t2 - t1, t3 - t2
        return {"t_iter": t_apply * self.scale_apply + t_patch * self.scale_patches + t_vec,
                "t_apply_sample": t_apply, "t_patches_sample": t_patch, "t_vector": t_vec,
                "scale_apply": self.scale_apply, "scale_patches": self.scale_patches,
                "sample_cells": int(len(self.cells)), "sample_patches": len(self.factors)}


class _Renumbered:
    """num.dofmap indexed by position in the sample's cell list (for _patch_matrix)."""

    def __init__(self, num, star_cells, cells):
        self.n_total = num.n_total
        self.dofmap = num.dofmap[cells]
