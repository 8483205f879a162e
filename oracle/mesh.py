"""Mesh topology, Dirichlet closure and the canonical global dof numbering.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:1279-1291: F_T preserves fixed global orientations of subsimplices; Dirichlet
dofs are removed by dropping the functions of entities on Gamma_D. DESIGN.md
readings R-A3 (sorted-vertex orientation), R-A9 (dimension-major numbering),
R-A11 (elimination; an entity is constrained iff it lies in the closure of a
Gamma_D face).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .simplex import TET_EDGES, TET_FACES


class MeshError(ValueError):
    pass


class Topology:
    def __init__(self, vertices, tets, mask):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        tets = np.asarray(tets, dtype=np.int64)
        self.tets_in = tets
        self.nv = self.vertices.shape[0]
        self.nt = tets.shape[0]
        self.cells = np.sort(tets, axis=1)          # F_T maps V-hat_k to the k-th smallest id
        # edges
        ce = np.stack([self.cells[:, [a, b]] for a, b in TET_EDGES], axis=1)  # [nt,6,2]
        self.edges, inv = np.unique(ce.reshape(-1, 2), axis=0, return_inverse=True)
        self.cell_edges = inv.reshape(self.nt, 6)
        cf = np.stack([self.cells[:, list(f)] for f in TET_FACES], axis=1)    # [nt,4,3]
        self.faces, inv, cnt = np.unique(cf.reshape(-1, 3), axis=0, return_inverse=True, return_counts=True)
        self.cell_faces = inv.reshape(self.nt, 4)
        if np.any(cnt > 2):
            raise MeshError("non-manifold face")
        self.boundary_face = cnt == 1
        self.ne, self.nf = len(self.edges), len(self.faces)
        # Dirichlet faces from the input-order mask
        mask = np.asarray(mask).astype(bool)
        dface = np.zeros(self.nf, dtype=bool)
        fidx = {tuple(f): i for i, f in enumerate(self.faces)}
        for t, i in zip(*np.nonzero(mask)):
            f = tuple(sorted(np.delete(tets[t], i)))
            fi = fidx[f]
            if not self.boundary_face[fi]:
                raise MeshError("Dirichlet mask bit set on an interior face")
            dface[fi] = True
        self.dir_face = dface
        self.dir_vertex = np.zeros(self.nv, dtype=bool)
        self.dir_vertex[self.faces[dface].ravel()] = True
        eidx = {tuple(e): i for i, e in enumerate(self.edges)}
        self.dir_edge = np.zeros(self.ne, dtype=bool)
        for f in self.faces[dface]:
            for a, b in ((0, 1), (0, 2), (1, 2)):
                self.dir_edge[eidx[(f[a], f[b])]] = True
        self.edge_index = eidx
        self.face_index = fidx
        # geometry check: |det J| > 1e-12 h^3
        x = self.vertices[self.cells]
        E = x[:, 1:] - x[:, :1]
        det = np.linalg.det(E)
        h = np.max(np.linalg.norm(E, axis=2), axis=1)
        if np.any(np.abs(det) <= 1e-12 * h ** 3):
            raise MeshError("degenerate tetrahedron")


def dof_layout(space: str, p: int):
    """Local dof list of T-hat, (dim, local entity, j, type) in the order of
    oracle.refelem (R-A8): vertices, edges (TET_EDGES), faces (TET_FACES), cell."""
    out = []
    if space == "hgrad":
        out += [(0, i, 0, "I") for i in range(4)]
        for dim, ne in ((1, 6), (2, 4), (3, 1)):
            nb = math.comb(p - 1, dim)
            out += [(dim, e, j, "I") for e in range(ne) for j in range(nb)]
        return out
    if space == "hdiv":  # RT_p (Eq. 3.18): face Whitney, face type-II, cell type-I, cell type-II
        nF = p * (p + 1) // 2 - 1
        nCI = p * (p + 1) * (p + 2) // 6 - 1
        nCII = p * (p - 1) * (p - 2) // 2 - (p - 1) * (p - 2) * (p - 3) // 6
        for e in range(4):
            out.append((2, e, 0, "W"))
            out += [(2, e, j, "II") for j in range(nF)]
        out += [(3, 0, j, "I") for j in range(nCI)]
        out += [(3, 0, j, "II") for j in range(nCII)]
        return out
    for e in range(6):
        out.append((1, e, 0, "W"))
        out += [(1, e, j, "II") for j in range(p - 1)]
    for dim, ne in ((2, 4), (3, 1)):
        nII = math.comb(p - 1, dim)
        nI = (p * (p - 1) if dim == 2 else p * (p - 1) * (p - 2) // 2) - nII
        for e in range(ne):
            out += [(dim, e, j, "I") for j in range(nI)]
            out += [(dim, e, j, "II") for j in range(nII)]
    return out


def dofs_per_entity(space: str, p: int):
    """(vertex, edge, face, cell) dof counts (Eq. 3.7)."""
    if space == "hgrad":
        return 1, p - 1, (p - 1) * (p - 2) // 2, (p - 1) * (p - 2) * (p - 3) // 6
    if space == "hdiv":
        return 0, 0, p * (p + 1) // 2, (p + 1) * p * (p - 1) // 2
    return 0, p, p * (p - 1), p * (p - 1) * (p - 2) // 2


@dataclass
class Numbering:
    """Global dofs, R-A9: [vertices][edges x ne_d][faces x nf_d][cells x nc_d]."""
    space: str
    p: int
    topo: Topology
    n_total: int
    offsets: tuple
    per: tuple
    dofmap: np.ndarray        # [nt, n_loc] global id of local dof
    constrained: np.ndarray   # bool [n_total]
    interior: np.ndarray      # bool [n_total] cell-interior dofs
    entity: np.ndarray        # [n_total, 2] (dim, entity id)
    kind: np.ndarray          # [n_total] "W"/"I"/"II"


def number(space: str, p: int, topo: Topology, dof_entity) -> Numbering:
    nvd, ned, nfd, ncd = dofs_per_entity(space, p)
    counts = (topo.nv * nvd, topo.ne * ned, topo.nf * nfd, topo.nt * ncd)
    offs = (0, counts[0], counts[0] + counts[1], counts[0] + counts[1] + counts[2])
    n_total = sum(counts)
    per = (nvd, ned, nfd, ncd)
    # within-entity position of each local dof (R-A8)
    nI_face = len([e for e in dof_entity if e[0] == 2 and e[1] == 0 and e[3] == "I"])
    nI_cell = len([e for e in dof_entity if e[0] == 3 and e[3] == "I"])
    n_loc = len(dof_entity)
    dofmap = np.zeros((topo.nt, n_loc), dtype=np.int64)
    for k, (dim, ei, j, typ) in enumerate(dof_entity):
        if dim == 0:
            ent = topo.cells[:, ei]
            pos = 0
        elif dim == 1:
            ent = topo.cell_edges[:, ei]
            pos = j if space == "hgrad" else (0 if typ == "W" else 1 + j)
        elif dim == 2:
            ent = topo.cell_faces[:, ei]
            if space == "hdiv":
                pos = 0 if typ == "W" else 1 + j
            else:
                pos = j if (space == "hgrad" or typ == "I") else nI_face + j
        else:
            ent = np.arange(topo.nt)
            pos = j if (space == "hgrad" or typ == "I") else nI_cell + j
        dofmap[:, k] = offs[dim] + ent * per[dim] + pos
    constrained = np.zeros(n_total, dtype=bool)
    interior = np.zeros(n_total, dtype=bool)
    entity = np.zeros((n_total, 2), dtype=np.int64)
    kind = np.empty(n_total, dtype=object)
    flags = (topo.dir_vertex, topo.dir_edge, topo.dir_face, np.zeros(topo.nt, dtype=bool))
    nents = (topo.nv, topo.ne, topo.nf, topo.nt)
    for dim in range(4):
        if per[dim] == 0:
            continue
        ids = offs[dim] + np.arange(nents[dim] * per[dim])
        constrained[ids] = np.repeat(flags[dim], per[dim])
        entity[ids, 0] = dim
        entity[ids, 1] = np.repeat(np.arange(nents[dim]), per[dim])
        if dim == 3:
            interior[ids] = True
    for k, (dim, ei, j, typ) in enumerate(dof_entity):
        kind[dofmap[:, k]] = typ
    return Numbering(space, p, topo, n_total, offs, per, dofmap, constrained, interior, entity, kind)
