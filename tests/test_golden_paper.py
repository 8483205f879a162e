"""Pins against values the paper prints (tests/golden/paper_patch_dimensions.txt,
each with its PAPER.md citation): the interior Freudenthal star counts, the
H(grad) vertex-star dimensions of §5.1 and every row of Table 1.

* The star counts are checked on an actual Freudenthal mesh (rdr_inputs).
* Every printed dimension is reproduced by counting the paper's dofs per
  entity (Eq. 3.7 / §3.4; type-I / type-II split Eq. 3.4-3.6) over
  the star -- this pins the dimension formulas the oracle and the library use.
* The rows this build implements (hgrad_interface_vertex; Eq. 5.12's
  ph_interface_typeI_J) are reproduced by the oracle's actual patch sets.
"""
import os

import numpy as np
import pytest

from rdr_inputs import make_config, HGRAD, HCURL
from oracle.solver import Oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_patch_dimensions.txt")


def _records():
    out = []
    for line in open(GOLDEN):
        line = line.split("#")[0].split()
        if line:
            out.append(line)
    return out


def _entries():
    return [r for r in _records() if r[0] != "star_counts"]


def cg(p):     # dofs per vertex / edge / face / cell, CG_p
    return 1, p - 1, (p - 1) * (p - 2) // 2, (p - 1) * (p - 2) * (p - 3) // 6


def ned(p):    # (total, type-I, type-II) per edge / face / cell, Ned1_p
    e = (p, 1, p - 1)
    f = (p * (p - 1), (p - 1) * (p + 2) // 2, (p - 1) * (p - 2) // 2)
    c = (p * (p - 1) * (p - 2) // 2, (p - 1) * (p - 2) * (2 * p + 3) // 6, (p - 1) * (p - 2) * (p - 3) // 6)
    return e, f, c


E_V, F_V, C_V = 14, 36, 24      # interior vertex star
F_E = C_E = 6                   # largest interior edge star: 6 faces, 6 cells (Table 1 caption P:2009-2010)


def rt(p):     # dofs per face / cell, RT_p (Eq. 3.18): face p(p+1)/2, cell p(p+1)(p-1)/2
    return p * (p + 1) // 2, (p + 1) * p * (p - 1) // 2


def counted_hdiv(label, p):
    """(vertex, edge, face) patch dims of Table 2's decompositions."""
    nf2, nc2 = rt(p)
    (ne1, _, _), (nf1, fI1, _), (nc1, _, _) = ned(p)
    return {"hdiv_pafw0_full": (F_V * nf2 + C_V * nc2, None, None),
            "hdiv_pafw0_interface_J": (F_V * nf2, None, None),
            "hdiv_ph_full": (None, ne1 + F_E * nf1 + C_E * nc1, nf2 + 2 * nc2),
            "hdiv_ph_typeI_interface_J": (None, 1 + F_E * fI1, None),
            "hdiv_pafw1_interface_J": (None, F_E * nf2, None)}[label]


def counted(label, p):
    if label.startswith("hdiv_"):
        return counted_hdiv(label, p)[:2]
    v, e, f, c = cg(p)
    (ne, _, _), (nf, fI, _), (nc, cI, _) = ned(p)
    vert = {"hgrad_full_vertex": v + E_V * e + F_V * f + C_V * c,
            "hgrad_interface_vertex": v + E_V * e + F_V * f,
            "pafw0_full": E_V * ne + F_V * nf + C_V * nc,
            "pafw0_interface_J": E_V * ne + F_V * nf,
            "ph_full": v + E_V * e + F_V * f + C_V * c,
            "ph_interface_J": v + E_V * e + F_V * f,
            "ph_typeI": v + E_V * e + F_V * f + C_V * c,
            "ph_interface_typeI_J": v + E_V * e + F_V * f}[label]
    edge = {"ph_full": ne + F_E * nf + C_E * nc,
            "ph_interface_J": ne + F_E * nf,
            "ph_typeI": 1 + F_E * fI + C_E * cI,
            "ph_interface_typeI_J": 1 + F_E * fI}.get(label)
    return vert, edge


def test_star_counts_on_freudenthal_mesh():
    rec = [r for r in _records() if r[0] == "star_counts"][0]
    n_e, n_f, n_c = (int(x) for x in rec[3:6])
    c = make_config(0, n=2, p=1, space=HGRAD, bc="none")
    o = Oracle(c.vertices, c.tets, 1, HGRAD, c.alpha, c.beta, c.mask, assemble=False)
    t = o.topo
    v = 1 + 3 * (1 + 3 * 1)  # the centre vertex (1,1,1) of the 2^3 mesh
    assert int(np.sum(np.any(t.edges == v, axis=1))) == n_e
    assert int(np.sum(np.any(t.faces == v, axis=1))) == n_f
    assert int(np.sum(np.any(t.cells == v, axis=1))) == n_c


@pytest.mark.parametrize("rec", _entries(), ids=lambda r: f"{r[0]}-p{r[2]}")
def test_printed_dimension_by_counting(rec):
    label, space, p, vdim, edim = rec[0], rec[1], int(rec[2]), rec[3], rec[4]
    v, e = counted(label, p)
    if vdim != "-":
        assert v == int(vdim)
    if edim != "-":
        assert e == int(edim)
    if len(rec) > 5:
        assert counted_hdiv(label, p)[2] == int(rec[5])


@pytest.mark.parametrize("p", [4, 10])
def test_implemented_rows_by_oracle_patches(p):
    recs = {(r[0], int(r[2])): r for r in _entries()}
    c = make_config(0, n=3, p=p, space=HGRAD, bc="none")
    o = Oracle(c.vertices, c.tets, p, HGRAD, c.alpha, c.beta, c.mask, assemble=False)
    assert max(len(i) for _, i in o.patch_sets()) == int(recs[("hgrad_interface_vertex", p)][3])
    o = Oracle(c.vertices, c.tets, p, HCURL, c.alpha, c.beta, c.mask, assemble=False)
    ps = o.patch_sets()
    r = recs[("ph_interface_typeI_J", p)]
    assert max(len(i) for k, i in ps if k == "pot") == int(r[3])
    assert max(len(i) for k, i in ps if k == "dof") == int(r[4])


@pytest.mark.parametrize("p", [4, 10])
def test_unsplit_rows_by_oracle_patches(p):
    """SURVEY NEXT-3 baselines: PAFW0(X0) (Eq. 5.2; P:1783-1786 prints 175 / 3439)
    and the type-I PH(X0, X1I) of Eq. 5.10 (Table 1 row ph_typeI: 175/121, 3439/1981)."""
    recs = {(r[0], int(r[2])): r for r in _entries()}
    c = make_config(0, n=3, p=p, space=HGRAD, bc="none")
    o = Oracle(c.vertices, c.tets, p, HGRAD, c.alpha, c.beta, c.mask, assemble=False, decomposition="unsplit")
    assert max(len(i) for _, i in o.patch_sets()) == int(recs[("hgrad_full_vertex", p)][3])
    o = Oracle(c.vertices, c.tets, p, HCURL, c.alpha, c.beta, c.mask, assemble=False, decomposition="unsplit")
    ps = o.patch_sets()
    r = recs[("ph_typeI", p)]
    assert max(len(i) for k, i in ps if k == "pot") == int(r[3])
    assert max(len(i) for k, i in ps if k == "dof") == int(r[4])


@pytest.mark.parametrize("p", [4, 10])
def test_hdiv_rows_by_oracle_patches(p):
    """the split H(div) decomposition PAFW1(X2_Gamma) + J(X2_I)
    (Eq. 5.16) has edge patches of Table 2's size (60 / 330), from the oracle's
    actual patch sets; the vertex-star interface/full counts of Table 2's
    PAFW0 rows (360 / 1980, 1080 / 13860) from its numbering."""
    recs = {(r[0], int(r[2])): r for r in _entries()}
    c = make_config(0, n=3, p=p, space=HGRAD, bc="none")
    o = Oracle(c.vertices, c.tets, p, "hdiv", c.alpha, c.beta, c.mask, assemble=False)
    ps = o.patch_sets()
    assert all(k == "dof" for k, _ in ps) and len(ps) == o.topo.ne
    assert max(len(i) for _, i in ps) == int(recs[("hdiv_pafw1_interface_J", p)][4])
    num, t = o.num, o.topo
    star_faces = max(int(np.sum(np.any(t.faces == v, axis=1))) for v in range(t.nv))
    star_cells = max(int(np.sum(np.any(t.cells == v, axis=1))) for v in range(t.nv))
    assert star_faces * num.per[2] == int(recs[("hdiv_pafw0_interface_J", p)][3])
    assert star_faces * num.per[2] + star_cells * num.per[3] == int(recs[("hdiv_pafw0_full", p)][3])
