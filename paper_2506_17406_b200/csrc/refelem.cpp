// Reference element of arXiv 2506.17406 on the equilateral T-hat, host side.
//
// Paper order: bubble spaces, augmented eigenproblem Eq. 3.9
// renormalised to Eq. 3.8, dofs of §3.4.1 Eq. 3.14
// and §3.4.2 Eq. 3.16, Ciarlet dual basis
// (P:883-900), reference matrices M-hat, K-hat^{ab}.
// Conventions: DESIGN.md R-A1..A8, R-A24, R-S1, R-S2. Everything is computed in
// x87 long double from exact barycentric integrals
//     int_S lambda^g = l! |S| g! / (|g| + l)!
// and rounded to double once at the end.
//
// Implementation choices (independent of the CPU oracle): pivoted Cholesky to
// extract a basis of a redundant spanning set, Cholesky reduction of the
// generalized problem, cyclic Jacobi for the symmetric eigenproblem, Gaussian
// elimination for the Vandermonde inverse.
#include "refelem.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <utility>

namespace rdr {
namespace {

typedef long double ld;

// ------------------------------------------------------------------ multi-indices
struct MI {
  int nv = 0, q = 0;
  std::vector<std::array<int, 4>> a;
  std::vector<int> lut;  // base-16 key -> index
  int key(const int* v) const {
    int k = 0;
    for (int i = nv - 1; i >= 0; --i) k = k * 16 + v[i];
    return k;
  }
  int find(const int* v) const { return lut[key(v)]; }
  int size() const { return (int)a.size(); }
};

std::mutex g_mi_mutex;
std::map<std::pair<int, int>, std::unique_ptr<MI>> g_mi;

void gen_mi(int nv, int q, int pos, std::array<int, 4>& cur, std::vector<std::array<int, 4>>& out) {
  if (pos == nv - 1) {
    cur[pos] = q;
    out.push_back(cur);
    return;
  }
  for (int v = 0; v <= q; ++v) {
    cur[pos] = v;
    gen_mi(nv, q - v, pos + 1, cur, out);
  }
}

const MI& mi(int nv, int q) {
  std::lock_guard<std::mutex> lk(g_mi_mutex);
  auto k = std::make_pair(nv, q);
  auto it = g_mi.find(k);
  if (it != g_mi.end()) return *it->second;
  auto m = std::make_unique<MI>();
  m->nv = nv;
  m->q = q;
  if (q >= 0) {
    std::array<int, 4> cur{0, 0, 0, 0};
    gen_mi(nv, q, 0, cur, m->a);
  }
  int sz = 1;
  for (int i = 0; i < nv; ++i) sz *= 16;
  m->lut.assign(sz, -1);
  for (int i = 0; i < (int)m->a.size(); ++i) m->lut[m->key(m->a[i].data())] = i;
  const MI& ref = *m;
  g_mi[k] = std::move(m);
  return ref;
}

ld fact(int k) {
  static ld t[64];
  static bool init = false;
  if (!init) {
    t[0] = 1;
    for (int i = 1; i < 64; ++i) t[i] = t[i - 1] * (ld)i;
    init = true;
  }
  return t[k];
}

long long multinom(const std::array<int, 4>& a, int nv) {
  int s = 0;
  for (int i = 0; i < nv; ++i) s += a[i];
  // exact in long double up to 13!
  ld r = fact(s);
  for (int i = 0; i < nv; ++i) r /= fact(a[i]);
  return (long long)llroundl(r);
}

// ------------------------------------------------------------------ dense long double matrices
struct Mat {
  int r = 0, c = 0;
  std::vector<ld> v;
  Mat() {}
  Mat(int r_, int c_) : r(r_), c(c_), v((size_t)r_ * c_, 0.0L) {}
  ld& operator()(int i, int j) { return v[(size_t)i * c + j]; }
  ld operator()(int i, int j) const { return v[(size_t)i * c + j]; }
  ld* row(int i) { return v.data() + (size_t)i * c; }
  const ld* row(int i) const { return v.data() + (size_t)i * c; }
};

Mat mul(const Mat& A, const Mat& B) {  // A B
  if (A.c != B.r) throw std::runtime_error("mul: shape");
  Mat C(A.r, B.c);
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < A.r; ++i) {
    ld* ci = C.row(i);
    const ld* ai = A.row(i);
    for (int k = 0; k < A.c; ++k) {
      ld a = ai[k];
      if (a == 0) continue;
      const ld* bk = B.row(k);
      for (int j = 0; j < B.c; ++j) ci[j] += a * bk[j];
    }
  }
  return C;
}

Mat mulT(const Mat& A, const Mat& B) {  // A B^T
  if (A.c != B.c) throw std::runtime_error("mulT: shape");
  Mat C(A.r, B.r);
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < A.r; ++i) {
    const ld* ai = A.row(i);
    for (int j = 0; j < B.r; ++j) {
      const ld* bj = B.row(j);
      ld s = 0;
      for (int k = 0; k < A.c; ++k) s += ai[k] * bj[k];
      C(i, j) = s;
    }
  }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j) T(j, i) = A(i, j);
  return T;
}

// ------------------------------------------------------------------ simplex geometry
struct Geo {
  int l = 0, nv = 0;
  ld x[4][3] = {};
  ld g[4][3] = {};   // Cartesian gradients of barycentrics
  ld G[4][4] = {};   // g_k . g_m
  ld vol = 0;
  int np = 0;
  int pa[6] = {}, pb[6] = {};
  ld H[6][6] = {};   // (g_a x g_b).(g_c x g_d)
  ld cr[6][3] = {};  // g_a x g_b (3D) or its scalar z-component in cr[.][0] (2D)
};

Geo make_geo(int l) {
  Geo S;
  S.l = l;
  S.nv = l + 1;
  const ld s3 = sqrtl(3.0L), s6 = sqrtl(6.0L);
  if (l == 1) {
    S.x[0][0] = -1;
    S.x[1][0] = 1;
  } else if (l == 2) {
    ld c[3][2] = {{-1, -1 / s3}, {1, -1 / s3}, {0, 2 / s3}};
    for (int i = 0; i < 3; ++i)
      for (int d = 0; d < 2; ++d) S.x[i][d] = c[i][d];
  } else {
    ld c[4][3] = {{-1, -1 / s3, -1 / s6}, {1, -1 / s3, -1 / s6}, {0, 2 / s3, -1 / s6}, {0, 0, 3 / s6}};
    for (int i = 0; i < 4; ++i)
      for (int d = 0; d < 3; ++d) S.x[i][d] = c[i][d];
  }
  // E[d][j] = x_{j+1}[d] - x_0[d]; invert by Gauss-Jordan
  ld E[3][6] = {};
  for (int d = 0; d < l; ++d) {
    for (int j = 0; j < l; ++j) E[d][j] = S.x[j + 1][d] - S.x[0][d];
    E[d][l + d] = 1;
  }
  ld det = 1;
  for (int k = 0; k < l; ++k) {
    int piv = k;
    for (int i = k + 1; i < l; ++i)
      if (fabsl(E[i][k]) > fabsl(E[piv][k])) piv = i;
    if (piv != k) {
      for (int j = 0; j < 2 * l; ++j) std::swap(E[k][j], E[piv][j]);
      det = -det;
    }
    ld d = E[k][k];
    det *= d;
    for (int j = 0; j < 2 * l; ++j) E[k][j] /= d;
    for (int i = 0; i < l; ++i)
      if (i != k) {
        ld f = E[i][k];
        for (int j = 0; j < 2 * l; ++j) E[i][j] -= f * E[k][j];
      }
  }
  // E^{-1}[j][d] = E[j][l+d]; grad lambda_{j+1} = row j of E^{-1}
  for (int j = 0; j < l; ++j)
    for (int d = 0; d < l; ++d) S.g[j + 1][d] = E[j][l + d];
  for (int d = 0; d < l; ++d) {
    ld s = 0;
    for (int j = 1; j <= l; ++j) s += S.g[j][d];
    S.g[0][d] = -s;
  }
  S.vol = fabsl(det) / fact(l);
  for (int a = 0; a < S.nv; ++a)
    for (int b = 0; b < S.nv; ++b) {
      ld s = 0;
      for (int d = 0; d < l; ++d) s += S.g[a][d] * S.g[b][d];
      S.G[a][b] = s;
    }
  S.np = 0;
  for (int a = 0; a < S.nv; ++a)
    for (int b = a + 1; b < S.nv; ++b) {
      S.pa[S.np] = a;
      S.pb[S.np] = b;
      ++S.np;
    }
  for (int i = 0; i < S.np; ++i)
    for (int j = 0; j < S.np; ++j) {
      int a = S.pa[i], b = S.pb[i], c = S.pa[j], d = S.pb[j];
      S.H[i][j] = S.G[a][c] * S.G[b][d] - S.G[a][d] * S.G[b][c];
    }
  for (int i = 0; i < S.np; ++i) {
    const ld* u = S.g[S.pa[i]];
    const ld* w = S.g[S.pb[i]];
    if (l == 3) {
      S.cr[i][0] = u[1] * w[2] - u[2] * w[1];
      S.cr[i][1] = u[2] * w[0] - u[0] * w[2];
      S.cr[i][2] = u[0] * w[1] - u[1] * w[0];
    } else if (l == 2) {
      S.cr[i][0] = u[0] * w[1] - u[1] * w[0];
    }
  }
  return S;
}

// I[i][j] = int_S lambda^(g_i + g_j)
Mat integrals(const Geo& S, int q1, int q2) {
  const MI& A = mi(S.nv, q1);
  const MI& B = mi(S.nv, q2);
  Mat I(A.size(), B.size());
  ld scale = fact(S.l) * S.vol / fact(q1 + q2 + S.l);
  for (int i = 0; i < A.size(); ++i)
    for (int j = 0; j < B.size(); ++j) {
      ld pr = 1;
      for (int k = 0; k < S.nv; ++k) pr *= fact(A.a[i][k] + B.a[j][k]);
      I(i, j) = pr * scale;
    }
  return I;
}

// Gram matrix of fields with nc components per monomial (layout [g][c]):
// out = sum_{c,c'} W[c][c'] A_c I B_c'^T
Mat gram(const Geo& S, const Mat& A, int qa, const Mat& B, int qb, int nc, const ld* W) {
  const int Na = mi(S.nv, qa).size(), Nb = mi(S.nv, qb).size();
  if (A.c != Na * nc || B.c != Nb * nc) throw std::runtime_error("gram: shape");
  Mat I = integrals(S, qa, qb);
  Mat out(A.r, B.r);
  std::vector<Mat> AI(nc);
  for (int c = 0; c < nc; ++c) {
    Mat Ac(A.r, Na);
    for (int i = 0; i < A.r; ++i)
      for (int g = 0; g < Na; ++g) Ac(i, g) = A(i, g * nc + c);
    AI[c] = mul(Ac, I);
  }
  for (int c2 = 0; c2 < nc; ++c2) {
    Mat AW(A.r, Nb);
    for (int c = 0; c < nc; ++c) {
      ld w = W[c * nc + c2];
      if (w == 0) continue;
      for (size_t k = 0; k < AW.v.size(); ++k) AW.v[k] += w * AI[c].v[k];
    }
    Mat Bc(B.r, Nb);
    for (int i = 0; i < B.r; ++i)
      for (int g = 0; g < Nb; ++g) Bc(i, g) = B(i, g * nc + c2);
    Mat P = mulT(AW, Bc);
    for (size_t k = 0; k < out.v.size(); ++k) out.v[k] += P.v[k];
  }
  return out;
}

Mat gram0(const Geo& S, const Mat& A, int qa, const Mat& B, int qb) {
  ld one = 1;
  return gram(S, A, qa, B, qb, 1, &one);
}
Mat gram1(const Geo& S, const Mat& A, int qa, const Mat& B, int qb) {
  ld W[16];
  for (int a = 0; a < S.nv; ++a)
    for (int b = 0; b < S.nv; ++b) W[a * S.nv + b] = S.G[a][b];
  return gram(S, A, qa, B, qb, S.nv, W);
}
Mat gram2(const Geo& S, const Mat& A, int qa, const Mat& B, int qb) {
  ld W[36];
  for (int a = 0; a < S.np; ++a)
    for (int b = 0; b < S.np; ++b) W[a * S.np + b] = S.H[a][b];
  return gram(S, A, qa, B, qb, S.np, W);
}

// ------------------------------------------------------------------ operators on field rows
// scalar deg q -> 1-form deg q-1: grad lambda^g = sum_m g_m lambda^(g - e_m) grad lambda_m
Mat apply_grad(const Mat& F, int nv, int q) {
  const MI& A = mi(nv, q);
  const MI& B = mi(nv, q - 1);
  Mat out(F.r, B.size() * nv);
  for (int g = 0; g < A.size(); ++g)
    for (int m = 0; m < nv; ++m) {
      if (A.a[g][m] == 0) continue;
      int b[4] = {A.a[g][0], A.a[g][1], A.a[g][2], A.a[g][3]};
      b[m] -= 1;
      int col = B.find(b) * nv + m;
      ld f = A.a[g][m];
      for (int i = 0; i < F.r; ++i) out(i, col) += f * F(i, g);
    }
  return out;
}

int pair_index(int nv, int a, int b) {  // a < b
  int k = 0;
  for (int i = 0; i < nv; ++i)
    for (int j = i + 1; j < nv; ++j) {
      if (i == a && j == b) return k;
      ++k;
    }
  return -1;
}

// 1-form deg q -> 2-form deg q-1: curl(lambda^g g_m) = sum_k g_k lambda^(g-e_k) g_k x g_m
Mat apply_curl(const Mat& F, int nv, int q) {
  const MI& A = mi(nv, q);
  const MI& B = mi(nv, q - 1);
  int np = nv * (nv - 1) / 2;
  Mat out(F.r, B.size() * np);
  for (int g = 0; g < A.size(); ++g)
    for (int m = 0; m < nv; ++m)
      for (int k = 0; k < nv; ++k) {
        if (k == m || A.a[g][k] == 0) continue;
        int b[4] = {A.a[g][0], A.a[g][1], A.a[g][2], A.a[g][3]};
        b[k] -= 1;
        ld sgn = (k < m) ? 1.0L : -1.0L;
        int col = B.find(b) * np + pair_index(nv, std::min(k, m), std::max(k, m));
        ld f = sgn * A.a[g][k];
        int src = g * nv + m;
        for (int i = 0; i < F.r; ++i) out(i, col) += f * F(i, src);
      }
  return out;
}

struct WElem {
  std::array<int, 4> a;
  int i, j;
};

// rows: (weight) lambda^alpha (lambda_i g_j - lambda_j g_i), |alpha| = q -> 1-form deg q+1
Mat whitney_rows(const std::vector<WElem>& el, int nv, int q, bool scaled) {
  const MI& B = mi(nv, q + 1);
  Mat out((int)el.size(), B.size() * nv);
  for (int r = 0; r < (int)el.size(); ++r) {
    ld w = scaled ? (ld)multinom(el[r].a, nv) : 1.0L;
    int ai[4] = {el[r].a[0], el[r].a[1], el[r].a[2], el[r].a[3]};
    int aj[4] = {ai[0], ai[1], ai[2], ai[3]};
    ai[el[r].i] += 1;
    aj[el[r].j] += 1;
    out(r, B.find(ai) * nv + el[r].j) += w;
    out(r, B.find(aj) * nv + el[r].i) -= w;
  }
  return out;
}

// trace onto the subsimplex s (parent nv = 4), child numbering = position in s
Mat trace(const Mat& F, int q, const int* s, int ns, bool oneform) {
  const MI& P = mi(4, q);
  const MI& C = mi(ns, q);
  int ncp = oneform ? 4 : 1, ncc = oneform ? ns : 1;
  Mat out(F.r, C.size() * ncc);
  for (int g = 0; g < P.size(); ++g) {
    bool ok = true;
    for (int k = 0; k < 4 && ok; ++k) {
      bool in = false;
      for (int t = 0; t < ns; ++t) in |= (s[t] == k);
      if (!in && P.a[g][k] != 0) ok = false;
    }
    if (!ok) continue;
    int cg[4] = {0, 0, 0, 0};
    for (int t = 0; t < ns; ++t) cg[t] = P.a[g][s[t]];
    int ci = C.find(cg);
    for (int t = 0; t < ncc; ++t) {
      int src = oneform ? g * ncp + s[t] : g;
      int dst = ci * ncc + t;
      for (int i = 0; i < F.r; ++i) out(i, dst) += F(i, src);
    }
  }
  return out;
}

ld monomial(const std::array<int, 4>& a, int nv, const ld* bary) {
  ld v = 1;
  for (int k = 0; k < nv; ++k)
    for (int e = 0; e < a[k]; ++e) v *= bary[k];
  return v;
}

ld eval0(const Mat& F, int r, const Geo& S, int q, const ld* bary) {
  const MI& A = mi(S.nv, q);
  ld s = 0;
  for (int g = 0; g < A.size(); ++g) s += F(r, g) * monomial(A.a[g], S.nv, bary);
  return s;
}

void eval1(const Mat& F, int r, const Geo& S, int q, const ld* bary, ld* out) {
  const MI& A = mi(S.nv, q);
  for (int d = 0; d < 3; ++d) out[d] = 0;
  for (int g = 0; g < A.size(); ++g) {
    ld mv = monomial(A.a[g], S.nv, bary);
    for (int m = 0; m < S.nv; ++m) {
      ld c = F(r, g * S.nv + m) * mv;
      for (int d = 0; d < S.l; ++d) out[d] += c * S.g[m][d];
    }
  }
}

// ------------------------------------------------------------------ 2-forms (RT_p)
struct W2Elem {
  std::array<int, 4> a;
  int i, j, k;
};

// rows: (weight) lambda^alpha (lambda_i g_j x g_k - lambda_j g_i x g_k + lambda_k g_i x g_j)
// on T-hat, |alpha| = q -> 2-form deg q+1 in the 6-pair frame
Mat whitney2_rows(const std::vector<W2Elem>& el, int q, bool scaled) {
  const MI& B = mi(4, q + 1);
  Mat out((int)el.size(), B.size() * 6);
  for (int r = 0; r < (int)el.size(); ++r) {
    const ld w = scaled ? (ld)multinom(el[r].a, 4) : 1.0L;
    const int term[3][3] = {{el[r].i, el[r].j, el[r].k}, {el[r].j, el[r].i, el[r].k}, {el[r].k, el[r].i, el[r].j}};
    const ld sgn[3] = {1, -1, 1};
    for (int t = 0; t < 3; ++t) {
      int a[4] = {el[r].a[0], el[r].a[1], el[r].a[2], el[r].a[3]};
      a[term[t][0]] += 1;
      out(r, B.find(a) * 6 + pair_index(4, term[t][1], term[t][2])) += sgn[t] * w;
    }
  }
  return out;
}

// 2-form deg q on T-hat -> scalar deg q-1:
// div(lambda^g g_a x g_b) = sum_k g_k lambda^(g - e_k) g_k . (g_a x g_b)
Mat apply_div(const Geo& T, const Mat& F, int q) {
  const MI& A = mi(4, q);
  const MI& B = mi(4, q - 1);
  Mat out(F.r, B.size());
  for (int g = 0; g < A.size(); ++g)
    for (int pr = 0; pr < 6; ++pr)
      for (int k = 0; k < 4; ++k) {
        if (A.a[g][k] == 0 || k == T.pa[pr] || k == T.pb[pr]) continue;
        int b[4] = {A.a[g][0], A.a[g][1], A.a[g][2], A.a[g][3]};
        b[k] -= 1;
        ld tp = 0;
        for (int d = 0; d < 3; ++d) tp += T.g[k][d] * T.cr[pr][d];
        const ld f = A.a[g][k] * tp;
        const int col = B.find(b), src = g * 6 + pr;
        for (int i = 0; i < F.r; ++i) out(i, col) += f * F(i, src);
      }
  return out;
}

// trace of 2-forms on T-hat onto the face s (sorted local vertices): the
// monomials supported on s and the pairs inside s, in the face's 3-pair frame
Mat trace2(const Mat& F, int q, const int* s) {
  const MI& P = mi(4, q);
  const MI& C = mi(3, q);
  Mat out(F.r, C.size() * 3);
  for (int g = 0; g < P.size(); ++g) {
    int cg[4] = {0, 0, 0, 0}, used = 0;
    for (int t = 0; t < 3; ++t) {
      cg[t] = P.a[g][s[t]];
      used += cg[t];
    }
    if (used != q) continue;  // some weight on the vertex off s
    const int ci = C.find(cg);
    for (int ta = 0; ta < 3; ++ta)
      for (int tb = ta + 1; tb < 3; ++tb) {
        const int src = g * 6 + pair_index(4, s[ta], s[tb]), dst = ci * 3 + pair_index(3, ta, tb);
        for (int i = 0; i < F.r; ++i) out(i, dst) += F(i, src);
      }
  }
  return out;
}

// 3D vector proxy of the 2-form row r at a barycentric point
void eval2(const Mat& F, int r, const Geo& T, int q, const ld* bary, ld* out) {
  const MI& A = mi(4, q);
  for (int d = 0; d < 3; ++d) out[d] = 0;
  for (int g = 0; g < A.size(); ++g) {
    const ld mv = monomial(A.a[g], 4, bary);
    for (int pr = 0; pr < 6; ++pr) {
      const ld c = F(r, g * 6 + pr) * mv;
      for (int d = 0; d < 3; ++d) out[d] += c * T.cr[pr][d];
    }
  }
}

// ------------------------------------------------------------------ dense solvers
// cyclic Jacobi: A = V diag(w) V^T, w ascending
void jacobi_eig(Mat A, std::vector<ld>& w, Mat& V) {
  const int n = A.r;
  V = Mat(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1;
  ld norm = 0;
  for (ld x : A.v) norm = std::max(norm, fabsl(x));
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotations = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const ld apq = A(p, q);
        if (apq == 0) continue;
        const ld app = A(p, p), aqq = A(q, q);
        if (fabsl(apq) <= 1e-22L * sqrtl(fabsl(app * aqq)) || fabsl(apq) <= 1e-32L * norm) {
          A(p, q) = A(q, p) = 0;
          continue;
        }
        ++rotations;
        ld theta = (aqq - app) / (2 * apq);
        ld t = (theta >= 0 ? 1.0L : -1.0L) / (fabsl(theta) + sqrtl(theta * theta + 1));
        ld c = 1 / sqrtl(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          ld akp = A(k, p), akq = A(k, q);
          ld np_ = c * akp - s * akq, nq = s * akp + c * akq;
          A(k, p) = A(p, k) = np_;
          A(k, q) = A(q, k) = nq;
        }
        A(p, p) = app - t * apq;
        A(q, q) = aqq + t * apq;
        A(p, q) = A(q, p) = 0;
        for (int k = 0; k < n; ++k) {
          ld vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * vkq;
          V(k, q) = s * vkp + c * vkq;
        }
      }
    if (rotations == 0) break;
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return A(a, a) < A(b, b); });
  w.resize(n);
  Mat Vs(n, n);
  for (int j = 0; j < n; ++j) {
    w[j] = A(ord[j], ord[j]);
    for (int i = 0; i < n; ++i) Vs(i, j) = V(i, ord[j]);
  }
  V = Vs;
}

// Symmetric eigendecomposition for the larger bubble problems: Householder
// reduction to tridiagonal form (accumulating the transformation), then the
// implicit QL iteration with Wilkinson shifts on the tridiagonal, rotations
// applied to the accumulated basis. O(n^3) with a small constant, where the
// cyclic Jacobi above needs ~10 sweeps of 6 n^3 (the RT_10 cell bubbles, n =
// 495, took most of a 36 s build). A = V diag(w) V^T, w ascending.
void tridiagonal_ql_eig(Mat A, std::vector<ld>& w, Mat& V) {
  const int n = A.r;
  std::vector<ld> d(n, 0), e(n, 0);
  // ---- Householder: A -> Q T Q^T, Q accumulated in A
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    ld h = 0;
    if (l > 0) {
      ld scale = 0;
      for (int k = 0; k <= l; ++k) scale += fabsl(A(i, k));
      if (scale == 0) {
        e[i] = A(i, l);
      } else {
        for (int k = 0; k <= l; ++k) {
          A(i, k) /= scale;
          h += A(i, k) * A(i, k);
        }
        ld f = A(i, l);
        ld g = f >= 0 ? -sqrtl(h) : sqrtl(h);
        e[i] = scale * g;
        h -= f * g;
        A(i, l) = f - g;
        f = 0;
        for (int j = 0; j <= l; ++j) {
          A(j, i) = A(i, j) / h;
          ld gg = 0;
          for (int k = 0; k <= j; ++k) gg += A(j, k) * A(i, k);
          for (int k = j + 1; k <= l; ++k) gg += A(k, j) * A(i, k);
          e[j] = gg / h;
          f += e[j] * A(i, j);
        }
        const ld hh = f / (h + h);
        for (int j = 0; j <= l; ++j) {
          const ld fj = A(i, j);
          const ld gj = e[j] - hh * fj;
          e[j] = gj;
          for (int k = 0; k <= j; ++k) A(j, k) -= fj * e[k] + gj * A(i, k);
        }
      }
    } else {
      e[i] = A(i, l);
    }
    d[i] = h;
  }
  d[0] = 0;
  e[0] = 0;
  for (int i = 0; i < n; ++i) {
    const int l = i - 1;
    if (d[i] != 0) {
#pragma omp parallel for schedule(static) if (l > 256)
      for (int j = 0; j <= l; ++j) {
        ld g = 0;
        for (int k = 0; k <= l; ++k) g += A(i, k) * A(k, j);
        for (int k = 0; k <= l; ++k) A(k, j) -= g * A(k, i);
      }
    }
    d[i] = A(i, i);
    A(i, i) = 1;
    for (int j = 0; j <= l; ++j) A(j, i) = A(i, j) = 0;
  }
  // ---- implicit QL on (d, e), rotations accumulated into the columns of A
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  if (n > 0) e[n - 1] = 0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const ld dd = fabsl(d[m]) + fabsl(d[m + 1]);
        if (fabsl(e[m]) <= LDBL_EPSILON * dd) break;
      }
      if (m != l) {
        if (iter++ == 100) throw std::runtime_error("tridiagonal QL did not converge");
        ld g = (d[l + 1] - d[l]) / (2 * e[l]);
        ld r = hypotl(g, 1.0L);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? fabsl(r) : -fabsl(r)));
        ld s = 1, c = 1, p = 0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          ld f = s * e[i];
          const ld b = c * e[i];
          r = hypotl(f, g);
          e[i + 1] = r;
          if (r == 0) {
            d[i + 1] -= p;
            e[m] = 0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < n; ++k) {
            f = A(k, i + 1);
            A(k, i + 1) = s * A(k, i) + c * f;
            A(k, i) = c * A(k, i) - s * f;
          }
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0;
      }
    } while (m != l);
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return d[a] < d[b]; });
  w.resize(n);
  V = Mat(n, n);
  for (int j = 0; j < n; ++j) {
    w[j] = d[ord[j]];
    for (int i = 0; i < n; ++i) V(i, j) = A(i, ord[j]);
  }
}

// pivoted Cholesky of a PSD Gram matrix: selected indices (pivot order) and the
// lower Cholesky factor L of M[sel][sel]
std::vector<int> pivoted_cholesky(const Mat& M, ld rel_tol, Mat& L) {
  const int n = M.r;
  Mat A = M;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  ld dmax0 = 0;
  for (int i = 0; i < n; ++i) dmax0 = std::max(dmax0, A(i, i));
  Mat Lf(n, n);
  int r = 0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (A(perm[i], perm[i]) > A(perm[piv], perm[piv])) piv = i;
    ld d = A(perm[piv], perm[piv]);
    if (d <= rel_tol * dmax0) break;
    std::swap(perm[k], perm[piv]);
    for (int j = 0; j < k; ++j) std::swap(Lf(k, j), Lf(piv, j));
    ld lkk = sqrtl(d);
    Lf(k, k) = lkk;
    int pk = perm[k];
    for (int i = k + 1; i < n; ++i) Lf(i, k) = A(perm[i], pk) / lkk;
    for (int i = k + 1; i < n; ++i) {
      int pi = perm[i];
      ld lik = Lf(i, k);
      for (int j = k + 1; j < n; ++j) A(pi, perm[j]) -= lik * Lf(j, k);
    }
    ++r;
  }
  L = Mat(r, r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j <= i; ++j) L(i, j) = Lf(i, j);
  return std::vector<int>(perm.begin(), perm.begin() + r);
}

// solve L X = B (L lower triangular) in place on B
void lower_solve(const Mat& L, Mat& B) {
  for (int col = 0; col < B.c; ++col)
    for (int i = 0; i < L.r; ++i) {
      ld s = B(i, col);
      for (int k = 0; k < i; ++k) s -= L(i, k) * B(k, col);
      B(i, col) = s / L(i, i);
    }
}
// solve L^T X = B in place
void upper_t_solve(const Mat& L, Mat& B) {
  for (int col = 0; col < B.c; ++col)
    for (int i = L.r - 1; i >= 0; --i) {
      ld s = B(i, col);
      for (int k = i + 1; k < L.r; ++k) s -= L(k, i) * B(k, col);
      B(i, col) = s / L(i, i);
    }
}

Mat cholesky_lower(const Mat& A) {  // A = L L^T, A SPD (long double)
  const int n = A.r;
  Mat L(n, n);
  for (int j = 0; j < n; ++j) {
    ld d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0)) throw std::runtime_error("cholesky: not SPD");
    L(j, j) = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      ld v = A(i, j);
      for (int k = 0; k < j; ++k) v -= L(i, k) * L(j, k);
      L(i, j) = v / L(j, j);
    }
  }
  return L;
}

Mat inverse(const Mat& M) {  // Gauss-Jordan with partial pivoting
  const int n = M.r;
  Mat A = M, X(n, n);
  for (int i = 0; i < n; ++i) X(i, i) = 1;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (fabsl(A(i, k)) > fabsl(A(piv, k))) piv = i;
    if (A(piv, k) == 0) throw std::runtime_error("singular Vandermonde");
    if (piv != k) {
      std::swap_ranges(A.row(k), A.row(k) + n, A.row(piv));
      std::swap_ranges(X.row(k), X.row(k) + n, X.row(piv));
    }
    ld d = A(k, k);
#pragma omp parallel for schedule(static)
    for (int i = k + 1; i < n; ++i) {
      ld f = A(i, k) / d;
      if (f == 0) continue;
      ld* ai = A.row(i);
      const ld* ak = A.row(k);
      for (int j = k; j < n; ++j) ai[j] -= f * ak[j];
      ld* xi = X.row(i);
      const ld* xk = X.row(k);
      for (int j = 0; j < n; ++j) xi[j] -= f * xk[j];
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    ld d = A(k, k);
    ld* xk = X.row(k);
    for (int j = 0; j < n; ++j) xk[j] /= d;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < k; ++i) {
      ld f = A(i, k);
      if (f == 0) continue;
      ld* xi = X.row(i);
      for (int j = 0; j < n; ++j) xi[j] -= f * xk[j];
    }
  }
  return X;
}

// ------------------------------------------------------------------ bubble eigenbases
struct Eig {
  std::vector<ld> mu, lam;
  Mat F;  // rows: psi_j (0-form deg p or 1-form deg p) on the canonical simplex
};

ld frac(ld x) { return x - floorl(x); }

void probe_point(int l, int i, ld* bary) {
  const ld th[4] = {sqrtl(2.0L) - 1, sqrtl(3.0L) - 1, sqrtl(5.0L) - 2, sqrtl(7.0L) - 2};
  ld s = 0;
  for (int k = 0; k <= l; ++k) {
    bary[k] = 1 + frac((ld)i * th[k]);
    s += bary[k];
  }
  for (int k = 0; k <= l; ++k) bary[k] /= s;
}

void probe_direction(int dim, int i, ld* u) {
  ld x = (ld)i;
  if (dim == 2) {
    u[0] = cosl(x);
    u[1] = sinl(x);
  } else {
    u[0] = sinl(2 * x) * cosl(x);
    u[1] = sinl(2 * x) * sinl(x);
    u[2] = cosl(2 * x);
  }
}

// R-A6: canonicalize clusters of equal eigenvalues and fix signs
// kind 0: 0-forms, 1: 1-forms, 2: 2-forms on T-hat (vector probe of the proxy)
void canonicalize(const Geo& S, int kind, int q, Eig& E) {
  const int n = (int)E.mu.size();
  int j = 0;
  while (j < n) {
    int c = 1;
    while (j + c < n && (E.mu[j + c] - E.mu[j + c - 1]) <= 1e-8L * E.mu[j + c]) ++c;
    ld rho = 0;
    for (int k = 0; k < c; ++k) rho = std::max(rho, sqrtl(E.lam[j + k] / S.vol));
    Mat P(c, c);
    for (int s = 0;; ++s) {
      if (s > 200) throw std::runtime_error("probe window search failed");
      for (int i = 0; i < c; ++i) {
        ld bary[4];
        probe_point(S.l, s + 1 + i, bary);
        for (int k = 0; k < c; ++k) {
          if (kind == 0) {
            P(i, k) = eval0(E.F, j + k, S, q, bary);
          } else {
            ld v[3], u[3];
            if (kind == 1)
              eval1(E.F, j + k, S, q, bary, v);
            else
              eval2(E.F, j + k, S, q, bary, v);
            probe_direction(S.l, s + 1 + i, u);
            ld d = 0;
            for (int t = 0; t < S.l; ++t) d += v[t] * u[t];
            P(i, k) = d;
          }
        }
      }
      // sigma_min(P) from the eigenvalues of P^T P
      Mat PtP(c, c);
      for (int a = 0; a < c; ++a)
        for (int b = 0; b < c; ++b) {
          ld sum = 0;
          for (int t = 0; t < c; ++t) sum += P(t, a) * P(t, b);
          PtP(a, b) = sum;
        }
      std::vector<ld> w;
      Mat V;
      jacobi_eig(PtP, w, V);
      ld smin = sqrtl(std::max(w[0], (ld)0));
      if (smin >= 1e-3L * rho) break;
    }
    // P^T = Q R (modified Gram-Schmidt, twice), psi <- psi Q
    Mat Pt = transpose(P), Q(c, c);
    for (int a = 0; a < c; ++a) {
      std::vector<ld> v(c);
      for (int t = 0; t < c; ++t) v[t] = Pt(t, a);
      for (int pass = 0; pass < 2; ++pass)
        for (int b = 0; b < a; ++b) {
          ld r = 0;
          for (int t = 0; t < c; ++t) r += Q(t, b) * v[t];
          for (int t = 0; t < c; ++t) v[t] -= r * Q(t, b);
        }
      ld nr = 0;
      for (int t = 0; t < c; ++t) nr += v[t] * v[t];
      nr = sqrtl(nr);
      for (int t = 0; t < c; ++t) Q(t, a) = v[t] / nr;
    }
    Mat blk(c, E.F.c);
    for (int a = 0; a < c; ++a)
      for (int col = 0; col < E.F.c; ++col) {
        ld s = 0;
        for (int t = 0; t < c; ++t) s += Q(t, a) * E.F(j + t, col);
        blk(a, col) = s;
      }
    for (int a = 0; a < c; ++a) std::copy(blk.row(a), blk.row(a) + E.F.c, E.F.row(j + a));
    j += c;
  }
}

// Eq. 3.9 on span(rows of Fspan), kernel dropped, renormalised to Eq. 3.8
Eig bubble_eigen(const Geo& S, int kind, const Mat& Fspan, int q, int dim_bubble, int n_kernel) {
  Mat M, K;
  if (kind == 0) {
    M = gram0(S, Fspan, q, Fspan, q);
    Mat dF = apply_grad(Fspan, S.nv, q);
    K = gram1(S, dF, q - 1, dF, q - 1);
  } else if (kind == 1) {
    M = gram1(S, Fspan, q, Fspan, q);
    Mat dF = apply_curl(Fspan, S.nv, q);
    K = gram2(S, dF, q - 1, dF, q - 1);
  } else {  // 2-forms on T-hat, d = div (Eq. 3.17)
    M = gram2(S, Fspan, q, Fspan, q);
    Mat dF = apply_div(S, Fspan, q);
    K = gram0(S, dF, q - 1, dF, q - 1);
  }
  Mat L;
  std::vector<int> sel = pivoted_cholesky(M, 1e-14L, L);
  if ((int)sel.size() != dim_bubble) throw std::runtime_error("bubble span rank mismatch");
  const int r = (int)sel.size();
  Mat Ks(r, r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) Ks(i, j) = K(sel[i], sel[j]);
  lower_solve(L, Ks);               // L^{-1} K
  Mat Kt = transpose(Ks);
  lower_solve(L, Kt);               // L^{-1} K L^{-T}
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < i; ++j) Kt(i, j) = Kt(j, i) = (Kt(i, j) + Kt(j, i)) / 2;
  std::vector<ld> mu;
  Mat Y;
  if (r > 64)
    tridiagonal_ql_eig(Kt, mu, Y);
  else
    jacobi_eig(Kt, mu, Y);
  ld mumax = mu.back();
  int nk = 0;
  while (nk < r && mu[nk] < 1e-8L * mumax) ++nk;
  if (nk != n_kernel) throw std::runtime_error("kernel dimension mismatch");
  upper_t_solve(L, Y);              // coefficients over the selected span rows
  Eig E;
  const int ne = r - nk;
  E.F = Mat(ne, Fspan.c);
  for (int j = 0; j < ne; ++j) {
    ld m = mu[nk + j];
    E.mu.push_back(m);
    E.lam.push_back(1 / m);
    ld sc = 1 / sqrtl(m);
    for (int k = 0; k < r; ++k) {
      ld c = Y(k, nk + j) * sc;
      if (c == 0) continue;
      const ld* fr = Fspan.row(sel[k]);
      ld* out = E.F.row(j);
      for (int col = 0; col < Fspan.c; ++col) out[col] += c * fr[col];
    }
  }
  canonicalize(S, kind, q, E);
  return E;
}

long long binom(int n, int k) {
  if (k < 0 || n < k) return 0;
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

std::mutex g_eig_mutex;
std::map<std::tuple<int, int, int>, std::unique_ptr<Eig>> g_eig;

const Eig& cg_bubbles(int l, int p) {
  {
    std::lock_guard<std::mutex> lk(g_eig_mutex);
    auto it = g_eig.find({0, l, p});
    if (it != g_eig.end()) return *it->second;
  }
  Geo S = make_geo(l);
  const MI& A = mi(l + 1, p);
  std::vector<int> rows;
  for (int g = 0; g < A.size(); ++g) {
    bool all = true;
    for (int k = 0; k <= l; ++k) all &= A.a[g][k] >= 1;
    if (all) rows.push_back(g);
  }
  auto E = std::make_unique<Eig>();
  int dim = (int)binom(p - 1, l);
  if (dim > 0) {
    Mat F((int)rows.size(), A.size());
    for (int r = 0; r < (int)rows.size(); ++r) F(r, rows[r]) = (ld)multinom(A.a[rows[r]], l + 1);
    *E = bubble_eigen(S, 0, F, p, dim, 0);
  } else {
    E->F = Mat(0, A.size());
  }
  std::lock_guard<std::mutex> lk(g_eig_mutex);
  const Eig& ref = *E;
  g_eig[{0, l, p}] = std::move(E);
  return ref;
}

const Eig& ned_bubbles(int l, int p) {
  {
    std::lock_guard<std::mutex> lk(g_eig_mutex);
    auto it = g_eig.find({1, l, p});
    if (it != g_eig.end()) return *it->second;
  }
  Geo S = make_geo(l);
  const int nv = l + 1;
  int dim = (l == 2) ? p * (p - 1) : p * (p - 1) * (p - 2) / 2;
  int nk = (int)binom(p - 1, l);
  auto E = std::make_unique<Eig>();
  if (dim > 0) {
    std::vector<WElem> el;
    const MI& A = mi(nv, p - 1);
    for (int i = 0; i < nv; ++i)
      for (int j = i + 1; j < nv; ++j)
        for (int g = 0; g < A.size(); ++g) {
          bool cov = true;
          for (int k = 0; k < nv; ++k)
            if (k != i && k != j && A.a[g][k] == 0) cov = false;
          if (cov) el.push_back({A.a[g], i, j});
        }
    Mat F = whitney_rows(el, nv, p - 1, true);
    *E = bubble_eigen(S, 1, F, p, dim, nk);
  } else {
    E->F = Mat(0, mi(nv, p).size() * nv);
  }
  std::lock_guard<std::mutex> lk(g_eig_mutex);
  const Eig& ref = *E;
  g_eig[{1, l, p}] = std::move(E);
  return ref;
}

// RT_p cell bubbles (Eq. 3.17): span {lambda^alpha w_ijk : supp(alpha) U {i,j,k} =
// all four vertices}, dim p(p+1)(p-1)/2, kernel = the divergence-free bubbles
const Eig& rt_bubbles(int p) {
  {
    std::lock_guard<std::mutex> lk(g_eig_mutex);
    auto it = g_eig.find({2, 3, p});
    if (it != g_eig.end()) return *it->second;
  }
  Geo T = make_geo(3);
  const int dim = p * (p + 1) * (p - 1) / 2, nI = p * (p + 1) * (p + 2) / 6 - 1;
  auto E = std::make_unique<Eig>();
  if (dim > 0 && nI > 0) {
    std::vector<W2Elem> el;
    const MI& A = mi(4, p - 1);
    const int faces[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};
    for (const auto& f : faces)
      for (int g = 0; g < A.size(); ++g) {
        bool cov = true;
        for (int k = 0; k < 4; ++k)
          if (k != f[0] && k != f[1] && k != f[2] && A.a[g][k] == 0) cov = false;
        if (cov) el.push_back({A.a[g], f[0], f[1], f[2]});
      }
    Mat F = whitney2_rows(el, p - 1, true);
    *E = bubble_eigen(T, 2, F, p, dim, dim - nI);
  } else {
    E->F = Mat(0, mi(4, p).size() * 6);
  }
  std::lock_guard<std::mutex> lk(g_eig_mutex);
  const Eig& ref = *E;
  g_eig[{2, 3, p}] = std::move(E);
  return ref;
}

// ------------------------------------------------------------------ elements
const int TET_EDGES[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
const int TET_FACES[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};

void append_rows(Mat& V, int& row, const Mat& Vs) {
  for (int i = 0; i < Vs.r; ++i) {
    std::copy(Vs.row(i), Vs.row(i) + Vs.c, V.row(row));
    ++row;
  }
}

std::unique_ptr<RefElement> build_cg(int p) {
  auto el = std::make_unique<RefElement>();
  el->space = 0;
  el->p = p;
  Geo T = make_geo(3);
  const MI& A = mi(4, p);
  const int n = A.size();
  el->n = n;
  Mat Span(n, n);  // scaled Bernstein (p!/b!) lambda^b
  for (int k = 0; k < n; ++k) Span(k, k) = (ld)multinom(A.a[k], 4);
  Mat V(n, n);
  int row = 0;
  for (int i = 0; i < 4; ++i) {  // vertex values
    int e[4] = {0, 0, 0, 0};
    e[i] = p;
    int col = A.find(e);
    for (int k = 0; k < n; ++k) V(row, k) = Span(k, col);
    el->dofs.push_back({0, i, 0, 0});
    ++row;
  }
  for (int dim = 1; dim <= 3; ++dim) {
    int nent = dim == 1 ? 6 : dim == 2 ? 4 : 1;
    const Eig& E = cg_bubbles(dim, p);
    if (E.mu.empty()) continue;
    Geo S = make_geo(dim);
    Mat gpsi = apply_grad(E.F, dim + 1, p);
    for (int e = 0; e < nent; ++e) {
      int s[4];
      if (dim == 1) { s[0] = TET_EDGES[e][0]; s[1] = TET_EDGES[e][1]; }
      else if (dim == 2) { for (int t = 0; t < 3; ++t) s[t] = TET_FACES[e][t]; }
      else { for (int t = 0; t < 4; ++t) s[t] = t; }
      Mat tr = trace(Span, p, s, dim + 1, false);
      Mat gv = apply_grad(tr, dim + 1, p);
      Mat Vs = gram1(S, gpsi, p - 1, gv, p - 1);
      append_rows(V, row, Vs);
      for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({dim, e, j, 0});
    }
  }
  if (row != n) throw std::runtime_error("CG dof count mismatch");
  Mat C = inverse(V);
  Mat Phi = mul(transpose(C), Span);  // rows = phi_j in monomial coefficients
  // reference matrices
  Mat Mh = gram0(T, Phi, p, Phi, p);
  Mat GP = apply_grad(Phi, 4, p);
  const int Np1 = mi(4, p - 1).size();
  std::vector<Mat> D(3, Mat(n, Np1));
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n; ++i)
      for (int g = 0; g < Np1; ++g) {
        ld s = 0;
        for (int m = 0; m < 4; ++m) s += GP(i, g * 4 + m) * T.g[m][a];
        D[a](i, g) = s;
      }
  Mat K[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b) K[a][b] = gram0(T, D[a], p - 1, D[b], p - 1);
  el->n_mat = 7;
  el->R.assign((size_t)7 * n * n, 0.0);
  auto put = [&](int s, auto f) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) el->R[((size_t)s * n + i) * n + j] = (double)f(i, j);
  };
  put(0, [&](int i, int j) { return Mh(i, j); });
  put(1, [&](int i, int j) { return K[0][0](i, j); });
  put(2, [&](int i, int j) { return K[1][1](i, j); });
  put(3, [&](int i, int j) { return K[2][2](i, j); });
  put(4, [&](int i, int j) { return K[0][1](i, j) + K[0][1](j, i); });
  put(5, [&](int i, int j) { return K[0][2](i, j) + K[0][2](j, i); });
  put(6, [&](int i, int j) { return K[1][2](i, j) + K[1][2](j, i); });
  for (ld l : cg_bubbles(3, p).lam) el->lam_cell.push_back((double)l);
  return el;
}

std::unique_ptr<RefElement> build_ned(int p) {
  auto el = std::make_unique<RefElement>();
  el->space = 1;
  el->p = p;
  Geo T = make_geo(3);
  std::vector<WElem> span;
  const MI& Am = mi(4, p - 1);
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j)
      for (int g = 0; g < Am.size(); ++g) {
        bool ok = true;
        for (int k = 0; k < i; ++k) ok &= Am.a[g][k] == 0;
        if (ok) span.push_back({Am.a[g], i, j});
      }
  const int n = (int)span.size();
  el->n = n;
  Mat Span = whitney_rows(span, 4, p - 1, true);  // 1-forms of degree p
  Mat V(n, n);
  int row = 0;
  for (int dim = 1; dim <= 3; ++dim) {
    int nent = dim == 1 ? 6 : dim == 2 ? 4 : 1;
    Geo S = make_geo(dim);
    const Eig& psi = cg_bubbles(dim, p);
    Mat gpsi = apply_grad(psi.F, dim + 1, p);
    Mat cPsi;
    if (dim >= 2) cPsi = apply_curl(ned_bubbles(dim, p).F, dim + 1, p);
    for (int e = 0; e < nent; ++e) {
      int s[4];
      if (dim == 1) { s[0] = TET_EDGES[e][0]; s[1] = TET_EDGES[e][1]; }
      else if (dim == 2) { for (int t = 0; t < 3; ++t) s[t] = TET_FACES[e][t]; }
      else { for (int t = 0; t < 4; ++t) s[t] = t; }
      Mat tr = trace(Span, p, s, dim + 1, true);
      if (dim == 1) {
        Mat t(1, 2);  // unit tangent from the lower to the higher vertex: g_1 - g_0
        t(0, 0) = -1;
        t(0, 1) = 1;
        Mat Vs = gram1(S, t, 0, tr, p);
        append_rows(V, row, Vs);
        el->dofs.push_back({1, e, 0, 2});
      } else if (cPsi.r > 0) {
        Mat cv = apply_curl(tr, dim + 1, p);
        Mat Vs = gram2(S, cPsi, p - 1, cv, p - 1);
        append_rows(V, row, Vs);
        for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({dim, e, j, 0});
      }
      if (gpsi.r > 0) {
        Mat Vs = gram1(S, gpsi, p - 1, tr, p);
        append_rows(V, row, Vs);
        for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({dim, e, j, 1});
      }
    }
  }
  if (row != n) throw std::runtime_error("Ned dof count mismatch");
  Mat C = inverse(V);
  Mat Phi = mul(transpose(C), Span);  // rows = phi_j as 1-forms of degree p
  const int Np = mi(4, p).size(), Np1 = mi(4, p - 1).size();
  std::vector<Mat> P(3, Mat(n, Np));
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n; ++i)
      for (int g = 0; g < Np; ++g) {
        ld s = 0;
        for (int m = 0; m < 4; ++m) s += Phi(i, g * 4 + m) * T.g[m][a];
        P[a](i, g) = s;
      }
  Mat CP = apply_curl(Phi, 4, p);
  std::vector<Mat> Rc(3, Mat(n, Np1));
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n; ++i)
      for (int g = 0; g < Np1; ++g) {
        ld s = 0;
        for (int k = 0; k < 6; ++k) s += CP(i, g * 6 + k) * T.cr[k][a];
        Rc[a](i, g) = s;
      }
  Mat Mm[3][3], Kk[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b) {
      Mm[a][b] = gram0(T, P[a], p, P[b], p);
      Kk[a][b] = gram0(T, Rc[a], p - 1, Rc[b], p - 1);
    }
  el->n_mat = 12;
  el->R.assign((size_t)12 * n * n, 0.0);
  auto put = [&](int s, const Mat& X, bool sym) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        el->R[((size_t)s * n + i) * n + j] = (double)(sym ? X(i, j) + X(j, i) : X(i, j));
  };
  const int ab[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  for (int a = 0; a < 3; ++a) put(a, Mm[a][a], false);
  for (int k = 0; k < 3; ++k) put(3 + k, Mm[ab[k][0]][ab[k][1]], true);
  for (int a = 0; a < 3; ++a) put(6 + a, Kk[a][a], false);
  for (int k = 0; k < 3; ++k) put(9 + k, Kk[ab[k][0]][ab[k][1]], true);
  for (ld l : ned_bubbles(3, p).lam) el->lam_cell.push_back((double)l);
  {  // factors through L2-orthonormal bases of P_p and P_{p-1} (RefElement::F)
    const Mat Lp = cholesky_lower(integrals(T, p, p));
    const Mat Lq = cholesky_lower(integrals(T, p - 1, p - 1));
    el->nfm = 3 * Np;
    el->nf = 3 * Np + 3 * Np1;
    el->F.assign((size_t)n * el->nf, 0.0);
    for (int a = 0; a < 3; ++a) {
      const Mat FM = mul(P[a], Lp), FK = mul(Rc[a], Lq);
      for (int i = 0; i < n; ++i) {
        for (int k = 0; k < Np; ++k) el->F[(size_t)i * el->nf + a * Np + k] = (double)FM(i, k);
        for (int k = 0; k < Np1; ++k) el->F[(size_t)i * el->nf + el->nfm + a * Np1 + k] = (double)FK(i, k);
      }
    }
  }
  return el;
}

// RT_p with the dofs of Eq. 3.18 per entity:
// face: Whitney (1, n.v)_F then type-II (curl_F Psi_{F,j}, n.v)_F; cell: type-I
// (div Phi_{C,j}, div v) then type-II (curl Psi_{C,j}, v), the Psi being the
// Ned1_p bubble eigenbases (DESIGN.md R-D1). Reference matrices: the 2-form
// proxy mass M^{ab} (6 symmetric combinations) and the div-div matrix.
std::unique_ptr<RefElement> build_rt(int p) {
  auto el = std::make_unique<RefElement>();
  el->space = 2;
  el->p = p;
  Geo T = make_geo(3), Fc = make_geo(2);
  std::vector<W2Elem> span;
  const MI& Am = mi(4, p - 1);
  const int faces[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};
  for (const auto& f : faces)
    for (int g = 0; g < Am.size(); ++g) {
      bool ok = true;
      for (int k = 0; k < f[0]; ++k) ok &= Am.a[g][k] == 0;
      if (ok) span.push_back({Am.a[g], f[0], f[1], f[2]});
    }
  const int n = (int)span.size();
  if (n != p * (p + 1) * (p + 3) / 2) throw std::runtime_error("RT span dimension mismatch");
  el->n = n;
  Mat Span = whitney2_rows(span, p - 1, true);  // 2-forms of degree p
  Mat V(n, n);
  int row = 0;
  Mat unit(1, 3);  // the constant face 2-form with proxy 1 (orientation of the sorted vertices)
  unit(0, pair_index(3, 0, 1)) = 1 / Fc.cr[pair_index(3, 0, 1)][0];
  const Eig& PsiF = ned_bubbles(2, p);
  Mat cPsiF;
  if (PsiF.F.r > 0) cPsiF = apply_curl(PsiF.F, 3, p);
  for (int e = 0; e < 4; ++e) {
    Mat tr = trace2(Span, p, faces[e]);
    append_rows(V, row, gram2(Fc, unit, 0, tr, p));
    el->dofs.push_back({2, e, 0, 2});
    if (cPsiF.r > 0) {
      Mat Vs = gram2(Fc, cPsiF, p - 1, tr, p);
      append_rows(V, row, Vs);
      for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({2, e, j, 1});
    }
  }
  Mat divSpan = apply_div(T, Span, p);
  const Eig& Phi = rt_bubbles(p);
  if (Phi.F.r > 0) {
    Mat Vs = gram0(T, apply_div(T, Phi.F, p), p - 1, divSpan, p - 1);
    append_rows(V, row, Vs);
    for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({3, 0, j, 0});
  }
  const Eig& PsiC = ned_bubbles(3, p);
  if (PsiC.F.r > 0) {
    Mat Vs = gram2(T, apply_curl(PsiC.F, 4, p), p - 1, Span, p);
    append_rows(V, row, Vs);
    for (int j = 0; j < Vs.r; ++j) el->dofs.push_back({3, 0, j, 1});
  }
  if (row != n) throw std::runtime_error("RT dof count mismatch");
  Mat C = inverse(V);
  Mat Phi2 = mul(transpose(C), Span);  // rows = phi_j as 2-forms of degree p
  const int Np = mi(4, p).size();
  std::vector<Mat> P(3, Mat(n, Np));
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n; ++i)
      for (int g = 0; g < Np; ++g) {
        ld s = 0;
        for (int k = 0; k < 6; ++k) s += Phi2(i, g * 6 + k) * T.cr[k][a];
        P[a](i, g) = s;
      }
  Mat D = apply_div(T, Phi2, p);
  Mat Mm[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b) Mm[a][b] = gram0(T, P[a], p, P[b], p);
  Mat Kd = gram0(T, D, p - 1, D, p - 1);
  el->n_mat = 7;
  el->R.assign((size_t)7 * n * n, 0.0);
  auto put = [&](int s, const Mat& X, bool sym) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        el->R[((size_t)s * n + i) * n + j] = (double)(sym ? X(i, j) + X(j, i) : X(i, j));
  };
  const int ab[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  for (int a = 0; a < 3; ++a) put(a, Mm[a][a], false);
  for (int k = 0; k < 3; ++k) put(3 + k, Mm[ab[k][0]][ab[k][1]], true);
  put(6, Kd, false);
  for (ld l : Phi.lam) el->lam_cell.push_back((double)l);
  {  // factors (RefElement::F): the proxy mass through P_p, the (scalar) divergence through P_{p-1}
    const Mat Lp = cholesky_lower(integrals(T, p, p));
    const Mat Lq = cholesky_lower(integrals(T, p - 1, p - 1));
    const int Np1 = mi(4, p - 1).size();
    el->nfm = 3 * Np;
    el->nf = 3 * Np + Np1;
    el->F.assign((size_t)n * el->nf, 0.0);
    const Mat FD = mul(D, Lq);
    for (int a = 0; a < 3; ++a) {
      const Mat FM = mul(P[a], Lp);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < Np; ++k) el->F[(size_t)i * el->nf + a * Np + k] = (double)FM(i, k);
    }
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < Np1; ++k) el->F[(size_t)i * el->nf + el->nfm + k] = (double)FD(i, k);
  }
  return el;
}

std::mutex g_el_mutex;
std::map<std::pair<int, int>, std::unique_ptr<RefElement>> g_el;

}  // namespace

// ---- on-disk cache: opt-in with RDR_CACHE_DIR. One file per
// (space, p): magic, sizes, the local dofs, R and lam_cell in FP64, then an
// FNV-1a checksum of everything before it. A file that does not validate is
// ignored (rebuilt and rewritten); writes go through a temporary + rename.
namespace {

constexpr char kCacheMagic[8] = {'R', 'D', 'R', 'R', 'E', 'F', '0', '2'};

uint64_t fnv1a(const std::string& b) {
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char c : b) h = (h ^ c) * 1099511628211ULL;
  return h;
}

template <class T>
void put(std::string& b, const T& v) {
  b.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <class T>
bool get(const std::string& b, size_t& at, T& v) {
  if (at + sizeof(T) > b.size()) return false;
  std::memcpy(&v, b.data() + at, sizeof(T));
  at += sizeof(T);
  return true;
}

std::string cache_path(int space, int p) {
  const char* dir = std::getenv("RDR_CACHE_DIR");
  if (!dir || !*dir) return std::string();
  return std::string(dir) + "/refelem_s" + std::to_string(space) + "_p" + std::to_string(p) + ".bin";
}

std::string serialize(const RefElement& el) {
  std::string b(kCacheMagic, 8);
  put(b, (int32_t)el.space);
  put(b, (int32_t)el.p);
  put(b, (int32_t)el.n);
  put(b, (int32_t)el.n_mat);
  put(b, (int64_t)el.dofs.size());
  for (const LocalDof& d : el.dofs) {
    put(b, (int32_t)d.dim);
    put(b, (int32_t)d.ent);
    put(b, (int32_t)d.j);
    put(b, (int32_t)d.type);
  }
  put(b, (int64_t)el.R.size());
  b.append(reinterpret_cast<const char*>(el.R.data()), sizeof(double) * el.R.size());
  put(b, (int64_t)el.lam_cell.size());
  b.append(reinterpret_cast<const char*>(el.lam_cell.data()), sizeof(double) * el.lam_cell.size());
  put(b, (int32_t)el.nf);
  put(b, (int32_t)el.nfm);
  b.append(reinterpret_cast<const char*>(el.F.data()), sizeof(double) * el.F.size());
  put(b, fnv1a(b));
  return b;
}

std::unique_ptr<RefElement> load_cached(int space, int p) {
  const std::string path = cache_path(space, p);
  if (path.empty()) return nullptr;
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return nullptr;
  std::string b;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) b.append(buf, got);
  std::fclose(f);
  if (b.size() < 16 || std::memcmp(b.data(), kCacheMagic, 8) != 0) return nullptr;
  uint64_t sum;
  std::memcpy(&sum, b.data() + b.size() - 8, 8);
  if (fnv1a(b.substr(0, b.size() - 8)) != sum) return nullptr;
  auto el = std::make_unique<RefElement>();
  size_t at = 8;
  int32_t sp, pp, n, nm;
  int64_t nd, nr, nlam;
  if (!get(b, at, sp) || !get(b, at, pp) || !get(b, at, n) || !get(b, at, nm) || !get(b, at, nd)) return nullptr;
  if (sp != space || pp != p || n <= 0 || nm <= 0 || nd != n) return nullptr;
  el->space = sp;
  el->p = pp;
  el->n = n;
  el->n_mat = nm;
  el->dofs.resize(nd);
  for (LocalDof& d : el->dofs) {
    int32_t v[4];
    for (int32_t& x : v)
      if (!get(b, at, x)) return nullptr;
    d = LocalDof{v[0], v[1], v[2], v[3]};
  }
  if (!get(b, at, nr) || nr != (int64_t)nm * n * n || at + 8 * nr > b.size()) return nullptr;
  el->R.resize(nr);
  std::memcpy(el->R.data(), b.data() + at, 8 * nr);
  at += 8 * nr;
  if (!get(b, at, nlam) || nlam < 0 || at + 8 * nlam > b.size()) return nullptr;
  el->lam_cell.resize(nlam);
  std::memcpy(el->lam_cell.data(), b.data() + at, 8 * nlam);
  at += 8 * nlam;
  int32_t nf, nfm;
  if (!get(b, at, nf) || !get(b, at, nfm) || nf < 0 || nfm < 0 || nfm > nf ||
      at + 8 * (size_t)nf * n + 8 != b.size())
    return nullptr;
  el->nf = nf;
  el->nfm = nfm;
  el->F.resize((size_t)nf * n);
  std::memcpy(el->F.data(), b.data() + at, 8 * (size_t)nf * n);
  return el;
}

void store_cached(const RefElement& el) {
  const std::string path = cache_path(el.space, el.p);
  if (path.empty()) return;
  const std::string tmp = path + ".tmp" + std::to_string((long long)std::rand());
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;  // the cache is best effort: an unwritable directory only costs the rebuild
  const std::string b = serialize(el);
  const bool ok = std::fwrite(b.data(), 1, b.size(), f) == b.size();
  if (std::fclose(f) != 0 || !ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
}

}  // namespace

const RefElement& reference_element(int space, int p) {
  std::lock_guard<std::mutex> lk(g_el_mutex);
  auto k = std::make_pair(space, p);
  auto it = g_el.find(k);
  if (it != g_el.end()) return *it->second;
  auto el = load_cached(space, p);
  if (!el) {
    el = space == 0 ? build_cg(p) : space == 1 ? build_ned(p) : build_rt(p);
    store_cached(*el);
  }
  const RefElement& ref = *el;
  g_el[k] = std::move(el);
  return ref;
}

std::vector<double> bubble_eigenvalues(int kind, int l, int p) {
  if (kind == 2 && l != 3) throw std::runtime_error("RT bubbles live on the cell");
  const Eig& E = kind == 0 ? cg_bubbles(l, p) : kind == 1 ? ned_bubbles(l, p) : rt_bubbles(p);
  std::vector<double> out;
  for (ld v : E.lam) out.push_back((double)v);
  return out;
}

}  // namespace rdr
