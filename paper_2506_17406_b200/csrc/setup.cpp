// Host setup: topology (R-A3, R-A9, R-A11), per-cell coefficients (Eq. 2.7
// pullbacks), star patches (R-A13, Eq. 5.4, Eq. 5.12
// P:1956-1970), patch inverses (R-A15) and the interior diagonal (R-A17).
#include "setup.hpp"
#include "dense.hpp"

#include <omp.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>

#include "../../include/rdr.h"

namespace rdr {

static const int kEdges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int kFaces[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};

static int local_edge(int a, int b) {  // a < b local vertices
  for (int e = 0; e < 6; ++e)
    if (kEdges[e][0] == a && kEdges[e][1] == b) return e;
  return -1;
}

int build_mesh(const double* x, int64_t nv, const int32_t* tets, int64_t nt, const uint8_t* mask, Mesh& m) {
  m.nv = nv;
  m.nt = nt;
  m.x.assign(x, x + 3 * nv);
  m.cells.resize(4 * nt);
  for (int64_t t = 0; t < nt; ++t) {
    int32_t v[4];
    for (int i = 0; i < 4; ++i) {
      v[i] = tets[4 * t + i];
      if (v[i] < 0 || v[i] >= nv) return RDR_EMESH;
    }
    std::sort(v, v + 4);
    for (int i = 0; i < 4; ++i) m.cells[4 * t + i] = v[i];
    if (v[0] == v[1] || v[1] == v[2] || v[2] == v[3]) return RDR_EMESH;
  }
  // edges, sorted lexicographically
  {
    struct K { int32_t a, b; int64_t slot; };
    std::vector<K> k(6 * nt);
    for (int64_t t = 0; t < nt; ++t)
      for (int e = 0; e < 6; ++e) k[6 * t + e] = {m.cells[4 * t + kEdges[e][0]], m.cells[4 * t + kEdges[e][1]], 6 * t + e};
    std::sort(k.begin(), k.end(), [](const K& p, const K& q) { return p.a != q.a ? p.a < q.a : (p.b != q.b ? p.b < q.b : p.slot < q.slot); });
    m.cell_edges.resize(6 * nt);
    m.edges.clear();
    for (size_t i = 0; i < k.size(); ++i) {
      if (i == 0 || k[i].a != k[i - 1].a || k[i].b != k[i - 1].b) {
        m.edges.push_back(k[i].a);
        m.edges.push_back(k[i].b);
      }
      m.cell_edges[k[i].slot] = (int32_t)(m.edges.size() / 2 - 1);
    }
    m.ne = (int64_t)m.edges.size() / 2;
  }
  std::vector<int32_t> fcount;
  {
    struct K { int32_t a, b, c; int64_t slot; };
    std::vector<K> k(4 * nt);
    for (int64_t t = 0; t < nt; ++t)
      for (int f = 0; f < 4; ++f)
        k[4 * t + f] = {m.cells[4 * t + kFaces[f][0]], m.cells[4 * t + kFaces[f][1]], m.cells[4 * t + kFaces[f][2]], 4 * t + f};
    std::sort(k.begin(), k.end(), [](const K& p, const K& q) {
      if (p.a != q.a) return p.a < q.a;
      if (p.b != q.b) return p.b < q.b;
      if (p.c != q.c) return p.c < q.c;
      return p.slot < q.slot;
    });
    m.cell_faces.resize(4 * nt);
    m.faces.clear();
    for (size_t i = 0; i < k.size(); ++i) {
      if (i == 0 || k[i].a != k[i - 1].a || k[i].b != k[i - 1].b || k[i].c != k[i - 1].c) {
        m.faces.push_back(k[i].a);
        m.faces.push_back(k[i].b);
        m.faces.push_back(k[i].c);
        fcount.push_back(0);
      }
      fcount.back() += 1;
      m.cell_faces[k[i].slot] = (int32_t)(m.faces.size() / 3 - 1);
    }
    m.nf = (int64_t)m.faces.size() / 3;
    for (int32_t c : fcount)
      if (c > 2) return RDR_EMESH;  // non-manifold
  }
  // Dirichlet faces from the input-order mask and their closure
  m.dir_v.assign(nv, 0);
  m.dir_e.assign(m.ne, 0);
  m.dir_f.assign(m.nf, 0);
  for (int64_t t = 0; t < nt; ++t)
    for (int i = 0; i < 4; ++i) {
      if (!mask[4 * t + i]) continue;
      int32_t v = tets[4 * t + i];
      int k = 0;
      while (m.cells[4 * t + k] != v) ++k;
      int lf = 3 - k;  // local face not containing sorted vertex k
      int32_t f = m.cell_faces[4 * t + lf];
      if (fcount[f] != 1) return RDR_EMESH;  // mask on an interior face
      m.dir_f[f] = 1;
    }
  for (int64_t t = 0; t < nt; ++t)
    for (int lf = 0; lf < 4; ++lf) {
      if (!m.dir_f[m.cell_faces[4 * t + lf]]) continue;
      for (int a = 0; a < 3; ++a) {
        m.dir_v[m.cells[4 * t + kFaces[lf][a]]] = 1;
        for (int b = a + 1; b < 3; ++b) m.dir_e[m.cell_edges[6 * t + local_edge(kFaces[lf][a], kFaces[lf][b])]] = 1;
      }
    }
  // degenerate cells: |det J| <= 1e-12 h^3
  for (int64_t t = 0; t < nt; ++t) {
    const double* p0 = &m.x[3 * m.cells[4 * t]];
    double E[3][3], h = 0;
    for (int k = 0; k < 3; ++k) {
      const double* pk = &m.x[3 * m.cells[4 * t + k + 1]];
      double l2 = 0;
      for (int d = 0; d < 3; ++d) {
        E[d][k] = pk[d] - p0[d];
        l2 += E[d][k] * E[d][k];
      }
      h = std::max(h, std::sqrt(l2));
    }
    double det = E[0][0] * (E[1][1] * E[2][2] - E[1][2] * E[2][1]) - E[0][1] * (E[1][0] * E[2][2] - E[1][2] * E[2][0]) +
                 E[0][2] * (E[1][0] * E[2][1] - E[1][1] * E[2][0]);
    if (!(std::fabs(det) > 1e-12 * h * h * h)) return RDR_EMESH;
  }
  return 0;
}

void build_numbering(const Mesh& m, const RefElement& el, Numbering& num) {
  const int p = el.p;
  num.space = el.space;
  num.p = p;
  if (el.space == 0) {
    num.per[0] = 1;
    num.per[1] = p - 1;
    num.per[2] = (int64_t)(p - 1) * (p - 2) / 2;
    num.per[3] = (int64_t)(p - 1) * (p - 2) * (p - 3) / 6;
  } else if (el.space == 1) {
    num.per[0] = 0;
    num.per[1] = p;
    num.per[2] = (int64_t)p * (p - 1);
    num.per[3] = (int64_t)p * (p - 1) * (p - 2) / 2;
  } else {  // RT_p (Eq. 3.18): dim P_{p-1}(F) per face, the bubbles per cell
    num.per[0] = 0;
    num.per[1] = 0;
    num.per[2] = (int64_t)p * (p + 1) / 2;
    num.per[3] = (int64_t)(p + 1) * p * (p - 1) / 2;
  }
  const int64_t cnt[4] = {m.nv * num.per[0], m.ne * num.per[1], m.nf * num.per[2], m.nt * num.per[3]};
  num.off[0] = 0;
  for (int d = 1; d < 4; ++d) num.off[d] = num.off[d - 1] + cnt[d - 1];
  num.n_total = num.off[3] + cnt[3];
  // within-entity positions (R-A8)
  int nI_face = 0, nI_cell = 0;
  for (const LocalDof& d : el.dofs) {
    if (d.dim == 2 && d.ent == 0 && d.type == 0) ++nI_face;
    if (d.dim == 3 && d.type == 0) ++nI_cell;
  }
  const int n = el.n;
  num.dofmap.resize((size_t)m.nt * n);
  for (int64_t t = 0; t < m.nt; ++t)
    for (int i = 0; i < n; ++i) {
      const LocalDof& d = el.dofs[i];
      int64_t ent, pos;
      if (d.dim == 0) {
        ent = m.cells[4 * t + d.ent];
        pos = 0;
      } else if (d.dim == 1) {
        ent = m.cell_edges[6 * t + d.ent];
        pos = el.space == 0 ? d.j : (d.type == 2 ? 0 : 1 + d.j);
      } else if (d.dim == 2) {
        ent = m.cell_faces[4 * t + d.ent];
        if (el.space == 2)  // face Whitney, then type-II
          pos = d.type == 2 ? 0 : 1 + d.j;
        else
          pos = (el.space == 0 || d.type == 0) ? d.j : nI_face + d.j;
      } else {
        ent = t;
        pos = (el.space == 0 || d.type == 0) ? d.j : nI_cell + d.j;
      }
      num.dofmap[(size_t)t * n + i] = (int32_t)(num.off[d.dim] + ent * num.per[d.dim] + pos);
    }
  num.constrained.assign(num.n_total, 0);
  const std::vector<uint8_t>* flags[3] = {&m.dir_v, &m.dir_e, &m.dir_f};
  for (int d = 0; d < 3; ++d) {
    if (num.per[d] == 0) continue;
    const auto& fl = *flags[d];
    for (size_t e = 0; e < fl.size(); ++e)
      if (fl[e])
        for (int64_t j = 0; j < num.per[d]; ++j) num.constrained[num.off[d] + e * num.per[d] + j] = 1;
  }
}

int build_entity_map(const Mesh& m, const Numbering& num, const RefElement& el, EntityMap& em) {
  // Under R-A3 / R-A9 every cell parametrises a shared entity identically, so
  // the global id of local dof i of cell t is base(t, entity of i) + pos(i),
  // with pos(i) the same on every cell; verified below against the dof map.
  const int n = el.n;
  auto local_entity = [](const LocalDof& d) { return d.dim == 0 ? d.ent : d.dim == 1 ? 4 + d.ent : d.dim == 2 ? 10 + d.ent : 14; };
  auto global_entity = [&](int64_t t, const LocalDof& d) -> int64_t {
    return d.dim == 0 ? m.cells[4 * t + d.ent] : d.dim == 1 ? m.cell_edges[6 * t + d.ent]
                                             : d.dim == 2 ? m.cell_faces[4 * t + d.ent] : t;
  };
  em.lut.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    const LocalDof& d = el.dofs[i];
    const int64_t pos = num.dofmap[i] - (num.off[d.dim] + global_entity(0, d) * num.per[d.dim]);
    if (pos < 0 || pos >= num.per[d.dim] || pos >= 512) return -1;
    em.lut[i] = (uint16_t)((local_entity(d) << 9) | pos);
  }
  const std::vector<uint8_t>* dir[4] = {&m.dir_v, &m.dir_e, &m.dir_f, nullptr};
  const int64_t nent[4] = {m.nv, m.ne, m.nf, m.nt};
  std::vector<int64_t> first[4];
  for (int d = 0; d < 4; ++d) first[d].assign(nent[d], -1);
  em.ebase.assign((size_t)m.nt * 16, -1);
  em.own.assign(m.nt, 0);
  static const int ldim[15] = {0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3};
  static const int lent[15] = {0, 1, 2, 3, 0, 1, 2, 3, 4, 5, 0, 1, 2, 3, 0};
  for (int64_t t = 0; t < m.nt; ++t)
    for (int le = 0; le < 15; ++le) {
      const int d = ldim[le];
      if (num.per[d] == 0) continue;
      LocalDof ld{d, lent[le], 0, 0};
      const int64_t g = global_entity(t, ld);
      const bool cons = dir[d] && (*dir[d])[g];
      if (!cons) em.ebase[(size_t)t * 16 + le] = (int32_t)(num.off[d] + g * num.per[d]);
      if (!cons && first[d][g] < 0) {
        first[d][g] = t;
        em.own[t] |= (uint16_t)(1u << le);
      }
    }
  for (int64_t t = 0; t < m.nt; ++t)
    for (int i = 0; i < n; ++i) {
      const int l = em.lut[i];
      const int32_t b = em.ebase[(size_t)t * 16 + (l >> 9)];
      const int32_t g = num.dofmap[(size_t)t * n + i];
      if (b < 0 ? !num.constrained[g] : (b + (l & 511) != g || num.constrained[g])) return -1;
    }
  return 0;
}

// J maps T-hat to the cell: J = E E-hat^{-1}, E columns x_k - x_0 (sorted vertices)
struct RefEdgeInverse {
  double Ehinv[3][3];
  RefEdgeInverse() {
    const double s3 = std::sqrt(3.0), s6 = std::sqrt(6.0);
    const double V[4][3] = {{-1, -1 / s3, -1 / s6}, {1, -1 / s3, -1 / s6}, {0, 2 / s3, -1 / s6}, {0, 0, 3 / s6}};
    double Eh[3][3];
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < 3; ++k) Eh[d][k] = V[k + 1][d] - V[0][d];
    double det = Eh[0][0] * (Eh[1][1] * Eh[2][2] - Eh[1][2] * Eh[2][1]) - Eh[0][1] * (Eh[1][0] * Eh[2][2] - Eh[1][2] * Eh[2][0]) +
                 Eh[0][2] * (Eh[1][0] * Eh[2][1] - Eh[1][1] * Eh[2][0]);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
        Ehinv[i][j] = (Eh[i1][j1] * Eh[i2][j2] - Eh[i1][j2] * Eh[i2][j1]) / det;
      }
  }
};

static void jacobian(const Mesh& m, int64_t t, double J[3][3]) {
  static const RefEdgeInverse ref;  // thread-safe initialisation
  const auto& Ehinv = ref.Ehinv;
  const double* p0 = &m.x[3 * m.cells[4 * t]];
  double E[3][3];
  for (int k = 0; k < 3; ++k) {
    const double* pk = &m.x[3 * m.cells[4 * t + k + 1]];
    for (int d = 0; d < 3; ++d) E[d][k] = pk[d] - p0[d];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += E[i][k] * Ehinv[k][j];
      J[i][j] = s;
    }
}

static void inv3(const double A[3][3], double B[3][3], double& det) {
  det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
        A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
      B[i][j] = (A[i1][j1] * A[i2][j2] - A[i1][j2] * A[i2][j1]) / det;
    }
}

// H(grad): c = (beta|J|, alpha G_xx, G_yy, G_zz, G_xy, G_xz, G_yz), G = |J| (J^T J)^{-1}
// H(curl): c = (beta GM_.. x6, alpha GK_.. x6), GM = |J| (J^T J)^{-1}, GK = J^T J / |J|
// H(div): c = (beta GK_.. x6, alpha / |J|) (phi = J phi-hat / det J, div phi = div-hat / det J)
// (Eq. 2.7: grad phi = J^{-T} grad-hat, phi = J^{-T} phi-hat, curl phi = J curl-hat / det J)
void cell_coefficients(const Mesh& m, int space, const double* alpha, const double* beta, std::vector<double>& c) {
  const int nm = space == 1 ? 12 : 7;
  c.assign((size_t)m.nt * nm, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < m.nt; ++t) {
    double J[3][3], JtJ[3][3], Inv[3][3], det, d2;
    jacobian(m, t, J);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += J[k][i] * J[k][j];
        JtJ[i][j] = s;
      }
    inv3(JtJ, Inv, d2);
    double Jinv[3][3];
    inv3(J, Jinv, det);
    const double aj = std::fabs(det);
    double* ct = &c[(size_t)t * nm];
    const int ii[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
    if (space == 0) {
      ct[0] = beta[t] * aj;
      for (int k = 0; k < 6; ++k) ct[1 + k] = alpha[t] * aj * Inv[ii[k][0]][ii[k][1]];
    } else if (space == 1) {
      for (int k = 0; k < 6; ++k) ct[k] = beta[t] * aj * Inv[ii[k][0]][ii[k][1]];
      for (int k = 0; k < 6; ++k) ct[6 + k] = alpha[t] * JtJ[ii[k][0]][ii[k][1]] / aj;
    } else {
      for (int k = 0; k < 6; ++k) ct[k] = beta[t] * JtJ[ii[k][0]][ii[k][1]] / aj;
      ct[6] = alpha[t] / aj;
    }
  }
}

void interior_inverse_diagonal(const Mesh& m, const Numbering& num, const RefElement& el,
                               const std::vector<double>& coef, std::vector<double>& dinv) {
  const int n = el.n, nm = el.n_mat;
  dinv.assign(num.n_total - num.off[3], 0.0);
  std::vector<int> loc;
  for (int i = 0; i < n; ++i)
    if (el.dofs[i].dim == 3) loc.push_back(i);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < m.nt; ++t)
    for (int i : loc) {
      double d = 0;
      for (int s = 0; s < nm; ++s) d += coef[(size_t)t * nm + s] * el.R[((size_t)s * n + i) * n + i];
      dinv[num.dofmap[(size_t)t * n + i] - num.off[3]] = 1.0 / d;
    }
}

void pack_patch_tiles(const double* W2, int n, double* out, PatchLayout layout) {
  // exact packed lower triangle in 32-row block rows (setup.hpp patch layout)
  const int nbk = (n + 31) / 32;
  for (int I = 0; I < nbk; ++I) {
    const int rows = std::min(32, n - 32 * I);
    for (int J = 0; J <= I; ++J) {
      double* tile = out + patch_tile_offset(n, I, J);
      if (J < I) {  // full-width tile, `rows` rows (setup.hpp layouts)
        for (int i = 0; i < rows; ++i)
          for (int kk = 0; kk < 32; ++kk)
            tile[layout == kTileGroups ? ((kk >> 2) * rows + i) * 4 + (kk & 3)
                                       : i * 32 + 2 * ((kk >> 1) ^ (i & 7)) + (kk & 1)] =
                W2[(size_t)(I * 32 + i) * n + J * 32 + kk];
      } else {      // diagonal: packed lower triangle by columns, (i,k), k<=i at k*rows - k(k-1)/2 + (i-k)
        for (int kk = 0; kk < rows; ++kk)
          for (int i = kk; i < rows; ++i) tile[kk * rows - kk * (kk - 1) / 2 + (i - kk)] = W2[(size_t)(I * 32 + i) * n + I * 32 + kk];
      }
    }
  }
}

int build_coarse(const Mesh& m, const Numbering& num, const RefElement& el, const std::vector<double>& coef,
                 std::vector<int32_t>& cidx, std::vector<double>& tiles, std::vector<double>* dense) {
  // W^k (Lemma 4.1): vertex dofs (H(grad)) / Whitney edge dofs (H(curl)) /
  // Whitney face dofs (H(div)), free ones
  const int n = el.n, nm = el.n_mat, wdim = num.space == 0 ? 0 : num.space == 1 ? 1 : 2;
  std::vector<int> loc;
  for (int i = 0; i < n; ++i)
    if (el.dofs[i].dim == wdim && (num.space == 0 || el.dofs[i].type == 2)) loc.push_back(i);
  std::vector<int32_t> pos(num.n_total, -1);
  cidx.clear();
  const int64_t first = num.off[wdim];
  const int64_t count = wdim == 0 ? m.nv : wdim == 1 ? m.ne : m.nf, stride = num.per[wdim];
  for (int64_t k = 0; k < count; ++k) {
    const int64_t g = first + k * stride;
    if (!num.constrained[g]) {
      pos[g] = (int32_t)cidx.size();
      cidx.push_back((int32_t)g);
    }
  }
  const int nc = (int)cidx.size();
  tiles.clear();
  if (nc == 0) return 0;
  std::vector<double> A((size_t)nc * nc, 0.0);
  for (int64_t t = 0; t < m.nt; ++t)
    for (int a : loc) {
      const int pa = pos[num.dofmap[(size_t)t * n + a]];
      if (pa < 0) continue;
      for (int b : loc) {
        const int pb = pos[num.dofmap[(size_t)t * n + b]];
        if (pb < 0) continue;
        double v = 0;
        for (int q = 0; q < nm; ++q) v += coef[(size_t)t * nm + q] * el.R[((size_t)q * n + a) * n + b];
        A[(size_t)pa * nc + pb] += v;
      }
    }
  if (dense) {  // the caller inverts on the device (patch_setup.cu dense_spd_inverse_packed)
    dense->swap(A);
    return 0;
  }
  std::vector<double> work;
  if (!spd_inverse(A.data(), nc, work)) return RDR_ENOTSPD;
  tiles.assign(patch_stored_doubles(nc), 0.0);
  pack_patch_tiles(A.data(), nc, tiles.data(), kTileGroups);
  return 0;
}

void build_gradient(const Mesh& m, const Numbering& ned, const Numbering& cg, Gradient& G) {
  const int64_t ncg = cg.n_total;
  std::vector<std::vector<std::pair<int32_t, double>>> rows(ncg);
  const int p = ned.p;
  for (int64_t e = 0; e < m.ne; ++e) {
    int32_t a = m.edges[2 * e], b = m.edges[2 * e + 1];
    int32_t w = (int32_t)(ned.off[1] + e * ned.per[1]);
    rows[a].push_back({w, -1.0});
    rows[b].push_back({w, +1.0});
    for (int j = 0; j < p - 1; ++j) rows[cg.off[1] + e * cg.per[1] + j].push_back({w + 1 + j, 1.0});
  }
  const int64_t nIf = ned.per[2] - cg.per[2], nIc = ned.per[3] - cg.per[3];
  for (int64_t f = 0; f < m.nf; ++f)
    for (int64_t j = 0; j < cg.per[2]; ++j)
      rows[cg.off[2] + f * cg.per[2] + j].push_back({(int32_t)(ned.off[2] + f * ned.per[2] + nIf + j), 1.0});
  for (int64_t t = 0; t < m.nt; ++t)
    for (int64_t j = 0; j < cg.per[3]; ++j)
      rows[cg.off[3] + t * cg.per[3] + j].push_back({(int32_t)(ned.off[3] + t * ned.per[3] + nIc + j), 1.0});
  G.ptr.assign(ncg + 1, 0);
  for (int64_t c = 0; c < ncg; ++c) G.ptr[c + 1] = G.ptr[c] + (int64_t)rows[c].size();
  G.col.resize(G.ptr[ncg]);
  G.val.resize(G.ptr[ncg]);
  for (int64_t c = 0; c < ncg; ++c)
    for (size_t k = 0; k < rows[c].size(); ++k) {
      G.col[G.ptr[c] + k] = rows[c][k].first;
      G.val[G.ptr[c] + k] = rows[c][k].second;
    }
}

// ---------------------------------------------------------------- patches
namespace {

struct CSR {
  std::vector<int64_t> ptr;
  std::vector<int32_t> ind;
};

CSR invert_incidence(int64_t nsrc, int64_t ntgt, int k, const std::vector<int32_t>& conn) {
  // conn: [nsrc][k] target ids -> CSR target -> list of src
  CSR c;
  c.ptr.assign(ntgt + 1, 0);
  for (int64_t s = 0; s < nsrc; ++s)
    for (int j = 0; j < k; ++j) c.ptr[conn[s * k + j] + 1]++;
  for (int64_t t = 0; t < ntgt; ++t) c.ptr[t + 1] += c.ptr[t];
  c.ind.resize(c.ptr[ntgt]);
  std::vector<int64_t> pos(c.ptr.begin(), c.ptr.end() - 1);
  for (int64_t s = 0; s < nsrc; ++s)
    for (int j = 0; j < k; ++j) c.ind[pos[conn[s * k + j]]++] = (int32_t)s;
  return c;
}

struct PatchDef {
  std::vector<int32_t> idx;    // sorted global ids
  std::vector<int32_t> cells;  // star cells
  int numbering;               // 0 own, 1 CG potential
};

// in-place Cholesky A = L L^T (row-major, lower), returns false if not SPD
}  // namespace

int build_patches(const Mesh& m, const Numbering& num, const RefElement& el, const std::vector<double>& coef,
                  const Numbering* cg_num, const RefElement* cg_el, const std::vector<double>* cg_coef,
                  Patches& P, PatchSink& sink, PatchLayout layout, bool unsplit, PatchAssembly* dev) {
  CSR v_cells = invert_incidence(m.nt, m.nv, 4, m.cells);
  CSR v_edges = invert_incidence(m.ne, m.nv, 2, m.edges);
  CSR v_faces = invert_incidence(m.nf, m.nv, 3, m.faces);
  std::vector<PatchDef> defs;
  auto star_dofs = [&](const Numbering& nb, int64_t v, std::vector<int32_t>& out) {
    if (nb.per[0] && !nb.constrained[nb.off[0] + v]) out.push_back((int32_t)(nb.off[0] + v));
    for (int64_t k = v_edges.ptr[v]; k < v_edges.ptr[v + 1]; ++k) {
      int64_t e = v_edges.ind[k];
      for (int64_t j = 0; j < nb.per[1]; ++j) {
        int64_t id = nb.off[1] + e * nb.per[1] + j;
        if (!nb.constrained[id]) out.push_back((int32_t)id);
      }
    }
    for (int64_t k = v_faces.ptr[v]; k < v_faces.ptr[v + 1]; ++k) {
      int64_t f = v_faces.ind[k];
      for (int64_t j = 0; j < nb.per[2]; ++j) {
        int64_t id = nb.off[2] + f * nb.per[2] + j;
        if (!nb.constrained[id]) out.push_back((int32_t)id);
      }
    }
  };
  for (int64_t v = 0; v < (num.space == 2 ? 0 : m.nv); ++v) {  // vertex stars (own dofs for H(grad), CG potential for H(curl))
    PatchDef d;
    d.numbering = num.space == 0 ? 0 : 1;
    const Numbering& vn = num.space == 0 ? num : *cg_num;
    star_dofs(vn, v, d.idx);
    if (unsplit)  // PAFW0(X) / PH(X0, .) (Eq. 5.2 / 5.10): the cells' interior dofs too
      for (int64_t k = v_cells.ptr[v]; k < v_cells.ptr[v + 1]; ++k)
        for (int64_t j = 0; j < vn.per[3]; ++j) d.idx.push_back((int32_t)(vn.off[3] + v_cells.ind[k] * vn.per[3] + j));
    if (d.idx.empty()) continue;
    std::sort(d.idx.begin(), d.idx.end());
    d.cells.assign(v_cells.ind.begin() + v_cells.ptr[v], v_cells.ind.begin() + v_cells.ptr[v + 1]);
    defs.push_back(std::move(d));
  }
  if (num.space >= 1) {  // edge stars: of the type-I space (H(curl)), of X^2_Gamma (H(div), Eq. 5.16)
    std::vector<int32_t> e_of_cell_edge = m.cell_edges;
    CSR e_cells = invert_incidence(m.nt, m.ne, 6, e_of_cell_edge);
    // face -> its 3 edges via the cells
    std::vector<int32_t> face_edges(3 * m.nf, -1);
    for (int64_t t = 0; t < m.nt; ++t)
      for (int lf = 0; lf < 4; ++lf) {
        int64_t f = m.cell_faces[4 * t + lf];
        int q = 0;
        for (int a = 0; a < 3; ++a)
          for (int b = a + 1; b < 3; ++b)
            face_edges[3 * f + q++] = m.cell_edges[6 * t + local_edge(kFaces[lf][a], kFaces[lf][b])];
      }
    CSR e_faces = invert_incidence(m.nf, m.ne, 3, face_edges);
    // H(curl): the face type-I dofs; H(div): every face dof (Whitney + type-II)
    const int64_t nIf = num.space == 2 ? num.per[2] : num.per[2] - (int64_t)(num.p - 1) * (num.p - 2) / 2;
    for (int64_t e = 0; e < m.ne; ++e) {
      PatchDef d;
      d.numbering = 0;
      if (num.space == 1) {
        int64_t w = num.off[1] + e * num.per[1];
        if (!num.constrained[w]) d.idx.push_back((int32_t)w);
      }
      for (int64_t k = e_faces.ptr[e]; k < e_faces.ptr[e + 1]; ++k) {
        int64_t f = e_faces.ind[k];
        for (int64_t j = 0; j < nIf; ++j) {
          int64_t id = num.off[2] + f * num.per[2] + j;
          if (!num.constrained[id]) d.idx.push_back((int32_t)id);
        }
      }
      if (unsplit) {  // PH(., X1I) (Eq. 5.10): the type-I dofs of the cells containing E too; PAFW1(X2): all
        const int64_t nIc =
            num.space == 2 ? num.per[3] : num.per[3] - (int64_t)(num.p - 1) * (num.p - 2) * (num.p - 3) / 6;
        for (int64_t k = e_cells.ptr[e]; k < e_cells.ptr[e + 1]; ++k)
          for (int64_t j = 0; j < nIc; ++j) d.idx.push_back((int32_t)(num.off[3] + e_cells.ind[k] * num.per[3] + j));
      }
      if (d.idx.empty()) continue;
      std::sort(d.idx.begin(), d.idx.end());
      d.cells.assign(e_cells.ind.begin() + e_cells.ptr[e], e_cells.ind.begin() + e_cells.ptr[e + 1]);
      defs.push_back(std::move(d));
    }
  }
  // order by decreasing size (stable)
  std::vector<int> order(defs.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return defs[a].idx.size() > defs[b].idx.size(); });
  const int64_t np = (int64_t)defs.size();
  P.n.resize(np);
  P.kind.resize(np);
  P.idx_off.assign(np + 1, 0);
  P.tile_off.assign(np + 1, 0);
  P.max_n = 0;
  P.alg_bytes = 0;
  for (int64_t k = 0; k < np; ++k) {
    const PatchDef& d = defs[order[k]];
    int n = (int)d.idx.size();
    int nb = (n + 31) / 32;
    P.n[k] = n;
    P.kind[k] = (uint8_t)d.numbering;
    P.idx_off[k + 1] = P.idx_off[k] + (int64_t)nb * 32;
    (void)nb;
    P.tile_off[k + 1] = P.tile_off[k] + patch_stored_doubles(n);
    P.max_n = std::max(P.max_n, n);
    P.alg_bytes += 8.0 * n * (n + 1) / 2;
  }
  P.total_doubles = P.tile_off[np];
  P.idx.assign(P.idx_off[np], -1);
  for (int64_t k = 0; k < np; ++k) std::copy(defs[order[k]].idx.begin(), defs[order[k]].idx.end(), P.idx.begin() + P.idx_off[k]);

  if (dev) {  // device setup: per patch, the (local dof, position) lists of its star cells
    std::vector<std::vector<int32_t>> cells(np), counts(np);
    std::vector<std::vector<uint32_t>> ents(np);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = 0; k < np; ++k) {
      const PatchDef& d = defs[order[k]];
      const Numbering& nb = d.numbering == 0 ? num : *cg_num;
      const int nl = d.numbering == 0 ? el.n : cg_el->n;
      for (int32_t t : d.cells) {
        int c = 0;
        for (int i = 0; i < nl; ++i) {
          const int32_t g = nb.dofmap[(size_t)t * nl + i];
          auto it = std::lower_bound(d.idx.begin(), d.idx.end(), g);
          if (it != d.idx.end() && *it == g) {
            ents[k].push_back(((uint32_t)i << 16) | (uint32_t)(it - d.idx.begin()));
            ++c;
          }
        }
        if (c) {
          cells[k].push_back(t);
          counts[k].push_back(c);
        }
      }
    }
    dev->rec_ptr.assign(np + 1, 0);
    for (int64_t k = 0; k < np; ++k) dev->rec_ptr[k + 1] = dev->rec_ptr[k] + (int64_t)cells[k].size();
    const int64_t nrec = dev->rec_ptr[np];
    dev->rec_cell.resize(nrec);
    dev->rec_off.assign(nrec + 1, 0);
    for (int64_t k = 0; k < np; ++k)
      for (size_t r = 0; r < cells[k].size(); ++r) {
        const int64_t g = dev->rec_ptr[k] + (int64_t)r;
        dev->rec_cell[g] = cells[k][r];
        dev->rec_off[g + 1] = dev->rec_off[g] + counts[k][r];
      }
    dev->ent.resize(dev->rec_off[nrec]);
    for (int64_t k = 0; k < np; ++k)
      std::copy(ents[k].begin(), ents[k].end(), dev->ent.begin() + dev->rec_off[dev->rec_ptr[k]]);
    return sink.reserve(P.total_doubles);
  }

  // assemble + invert + pack, in chunks of about 1 GiB of tiles
  const int64_t chunk_doubles = std::max<int64_t>((int64_t)1 << 27, P.tile_off[1] - P.tile_off[0]);
  std::vector<double> buf;
  int status = sink.reserve(P.total_doubles);
  int64_t k0 = 0;
  while (k0 < np && status == 0) {
    int64_t k1 = k0;
    while (k1 < np && (P.tile_off[k1 + 1] - P.tile_off[k0] <= chunk_doubles || k1 == k0)) ++k1;
    const int64_t base = P.tile_off[k0];
    buf.assign(P.tile_off[k1] - base, 0.0);
#pragma omp parallel
    {
      std::vector<double> A, W1;
      std::vector<int> lpos;
#pragma omp for schedule(dynamic, 1)
      for (int64_t k = k0; k < k1; ++k) {
        if (status) continue;
        const PatchDef& d = defs[order[k]];
        const int n = (int)d.idx.size();
        const Numbering& nb = d.numbering == 0 ? num : *cg_num;
        const RefElement& re = d.numbering == 0 ? el : *cg_el;
        const std::vector<double>& cf = d.numbering == 0 ? coef : *cg_coef;
        const int nl = re.n, nm = re.n_mat;
        A.assign((size_t)n * n, 0.0);
        for (int32_t t : d.cells) {
          lpos.assign(nl, -1);
          std::vector<int> li;
          for (int i = 0; i < nl; ++i) {
            int32_t g = nb.dofmap[(size_t)t * nl + i];
            auto it = std::lower_bound(d.idx.begin(), d.idx.end(), g);
            if (it != d.idx.end() && *it == g) {
              lpos[i] = (int)(it - d.idx.begin());
              li.push_back(i);
            }
          }
          const double* c = &cf[(size_t)t * nm];
          for (int a : li)
            for (int b : li) {
              double s = 0;
              for (int q = 0; q < nm; ++q) s += c[q] * re.R[((size_t)q * nl + a) * nl + b];
              A[(size_t)lpos[a] * n + lpos[b]] += s;
            }
        }
        if (!spd_inverse(A.data(), n, W1)) {
#pragma omp atomic write
          status = RDR_ENOTSPD;
          continue;
        }
        const std::vector<double>& W2 = A;  // A^-1, both triangles
        pack_patch_tiles(W2.data(), n, buf.data() + (P.tile_off[k] - base), layout);
      }
    }
    if (status) break;
    status = sink.put(base, buf.data(), (int64_t)buf.size());
    k0 = k1;
  }
  return status;
}

}  // namespace rdr
