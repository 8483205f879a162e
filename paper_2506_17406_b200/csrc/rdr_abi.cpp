// C ABI of the library (include/rdr.h): host setup once, then device-resident
// operator, preconditioner and PCG.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <mutex>
#include <set>
#include <vector>

#include "../../include/rdr.h"
#include "kernels.hpp"
#include "refelem.hpp"
#include "setup.hpp"
#include "dense.hpp"
#include "patch_setup.hpp"

using namespace rdr;

namespace {

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RDR_OK;
  if (e == cudaErrorMemoryAllocation) return RDR_ENOMEM;
  return RDR_ECUDA;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      std::fprintf(stderr, "rdr: %s (%s:%d)\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return cuda_status(e_);                                                                 \
    }                                                                                         \
  } while (0)

template <class T>
int upload(T** dptr, const std::vector<T>& h) {
  *dptr = nullptr;
  if (h.empty()) return RDR_OK;
  CK(cudaMalloc((void**)dptr, sizeof(T) * h.size()));
  CK(cudaMemcpy(*dptr, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return RDR_OK;
}

// copy a caller array (host or device) into a host vector
template <class T>
int fetch(const T* p, size_t count, std::vector<T>& out) {
  out.resize(count);
  if (count == 0) return RDR_OK;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    a.type = cudaMemoryTypeUnregistered;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    CK(cudaMemcpy(out.data(), p, sizeof(T) * count, cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(out.data(), p, sizeof(T) * count);
  }
  return RDR_OK;
}

struct DeviceTiles : PatchSink {
  double* d = nullptr;
  int reserve(int64_t total) override {
    if (total == 0) return RDR_OK;
    cudaError_t e = cudaMalloc((void**)&d, sizeof(double) * total);
    return cuda_status(e);
  }
  int put(int64_t begin, const double* tiles, int64_t count) override {
    cudaError_t e = cudaMemcpy(d + begin, tiles, sizeof(double) * count, cudaMemcpyHostToDevice);
    return cuda_status(e);
  }
};

// uniform[-1,1] from splitmix64(seed + i) (the counter-based Lanczos start
// vector of the hybrid weights; oracle/hybrid.py lanczos_rhs implements the same)
double splitmix_uniform(uint64_t seed, uint64_t i) {
  uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}
constexpr uint64_t kLanczosSeed = 0x5EED;
constexpr int kLanczosSteps = 10;

// eigenvalues of a small symmetric matrix (cyclic Jacobi), ascending
std::vector<double> sym_eigenvalues(std::vector<double> A, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double theta = (A[q * n + q] - A[p * n + p]) / (2 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), sn = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - sn * akq;
          A[k * n + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - sn * aqk;
          A[q * n + k] = sn * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
  std::sort(ev.begin(), ev.end());
  return ev;
}

// The persisting-L2 set-aside is a device-wide limit: handles that hold a
// window register their size here; the limit is the largest registered size
// and is reset (with the persisting lines) only when the last owner goes.
std::mutex g_l2_mutex;
std::multiset<size_t> g_l2_owners;

void l2_window_acquire(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_l2_mutex);
  g_l2_owners.insert(bytes);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, *g_l2_owners.rbegin());
  cudaGetLastError();
}

void l2_window_release(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_l2_mutex);
  auto it = g_l2_owners.find(bytes);
  if (it != g_l2_owners.end()) g_l2_owners.erase(it);
  if (g_l2_owners.empty()) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  } else {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, *g_l2_owners.rbegin());
  }
  cudaGetLastError();
}

}  // namespace

struct rdr_handle {
  int space = 0, p = 0;
  int64_t n_total = 0;
  rdr_info info{};
  DevOperator op{};
  DevPrecond pc{};
  // owned device memory
  std::vector<void*> owned;
  uint8_t* d_cons = nullptr;
  double *d_x = nullptr, *d_r = nullptr, *d_z = nullptr, *d_p = nullptr, *d_q = nullptr, *d_b = nullptr;
  double* d_p2 = nullptr;  // second search-direction buffer of the fused path
  bool fused = false;
  cudaAccessPolicyWindow l2_window{};  // persisting window over the PCG slab (num_bytes 0: none)
  PcgScalars* d_sc = nullptr;
  PcgScalars* h_sc = nullptr;  // pinned
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t wgraph = nullptr;  // device-side while loop (fused path)
  int loop = RDR_LOOP_DEVICE;        // rdr_options.loop
  PersistentPcg persist;             // the persistent PCG kernel's plan (grid 0: not eligible)
  bool use_persist = false;          // solves run as one persistent cooperative launch
  int graph_iters = 0;
  int launches_per_iter = 0;
  double rho1 = 1.0, rho2 = 1.0;  // hybrid Schwarz weights (rdr_get_weights)
  int64_t last_launches = 0;

  template <class T>
  int own_upload(T** d, const std::vector<T>& h) {
    int st = upload(d, h);
    if (*d) owned.push_back((void*)*d);
    return st;
  }
  int own_alloc(void** d, size_t bytes) {
    CK(cudaMalloc(d, bytes));
    owned.push_back(*d);
    return RDR_OK;
  }
  ~rdr_handle() {
    if (graph) cudaGraphExecDestroy(graph);
    if (wgraph) cudaGraphExecDestroy(wgraph);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (l2_window.num_bytes) l2_window_release(l2_window.num_bytes);
    for (void* p : owned) cudaFree(p);
    if (h_sc) cudaFreeHost(h_sc);
  }
};

static int hybrid_weights(rdr_handle* h, const std::vector<double>& dinv);
static int select_loop(rdr_handle* h);

// device memory freed at scope exit (setup temporaries)
struct DevTemps {
  std::vector<void*> p;
  template <class T>
  int up(const T** d, const std::vector<T>& h) {
    T* q = nullptr;
    const int st = upload(&q, h);
    if (q) p.push_back(q);
    *d = q;
    return st;
  }
  ~DevTemps() {
    for (void* q : p) cudaFree(q);
  }
};

// Assemble, invert and pack every patch on the GPU (SURVEY NEXT-4,
// patch_setup.cu) into the already reserved store s.tiles.
static int device_patch_setup(DevPatchSetup s, const Patches& P, const PatchAssembly& pa, const RefElement* cg_el,
                              const std::vector<double>* cg_coef, double* kernel_seconds) {
  DevTemps tmp;
  int st;
  if ((st = tmp.up(&s.rec_ptr, pa.rec_ptr))) return st;
  if ((st = tmp.up(&s.rec_cell, pa.rec_cell))) return st;
  if ((st = tmp.up(&s.rec_off, pa.rec_off))) return st;
  if ((st = tmp.up(&s.ent, pa.ent))) return st;
  if (cg_el) {
    if ((st = tmp.up(&s.R[1], cg_el->R))) return st;
    if ((st = tmp.up(&s.coef[1], *cg_coef))) return st;
    s.nl[1] = cg_el->n;
    s.nm[1] = cg_el->n_mat;
  }
  s.np = (int64_t)P.n.size();
  s.ld_max = (P.max_n + 63) / 64 * 64;
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  // scratch: two CTAs per SM, within min(16 GiB, half the free memory)
  const double per_cta = 8.0 * (double)patch_setup_scratch_doubles(s.ld_max);
  const double budget = std::min(16.0 * (1 << 30), 0.5 * (double)free_b);
  const int ctas = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)2 * sms, s.np, (int64_t)(budget / per_cta)}));
  double* scratch = nullptr;
  CK(cudaMalloc((void**)&scratch, (size_t)per_cta * ctas));
  tmp.p.push_back(scratch);
  int32_t* ctl = nullptr;
  CK(cudaMalloc((void**)&ctl, 2 * sizeof(int32_t)));
  tmp.p.push_back(ctl);
  CK(cudaMemset(ctl, 0, 2 * sizeof(int32_t)));
  s.scratch = scratch;
  s.queue = ctl;
  s.status = ctl + 1;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, 0));
  CK(launch_patch_setup(s, ctas, 0));
  CK(cudaEventRecord(e1, 0));
  int32_t status = 0;
  CK(cudaMemcpy(&status, s.status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *kernel_seconds = 1e-3 * ms;
  return status ? RDR_ENOTSPD : RDR_OK;
}

static int setup_impl(rdr_handle* h, const double* vertices, int64_t nv, const int32_t* tets, int64_t nt, int p,
                      int space, const double* alpha, const double* beta, const uint8_t* mask, bool unsplit,
                      bool hybrid, bool host_setup, int loop, cudaStream_t stream) {
  auto t0 = std::chrono::steady_clock::now();
  if (stream) CK(cudaStreamSynchronize(stream));
  configure_kernels();
  std::vector<double> hx, ha, hb;
  std::vector<int32_t> ht;
  std::vector<uint8_t> hm;
  int st;
  if ((st = fetch(vertices, (size_t)nv * 3, hx))) return st;
  if ((st = fetch(tets, (size_t)nt * 4, ht))) return st;
  if ((st = fetch(alpha, (size_t)nt, ha))) return st;
  if ((st = fetch(beta, (size_t)nt, hb))) return st;
  if ((st = fetch(mask, (size_t)nt * 4, hm))) return st;
  // alpha > 0, beta >= 0; H(curl) and H(div) need beta > 0: with beta = 0
  // gradients (curl-free fields) resp. div-free fields are in the kernel of A and
  // of the star-patch matrices (their tiny rounded pivots would not be caught)
  for (int64_t t = 0; t < nt; ++t)
    if (!(ha[t] > 0) || !(hb[t] >= 0) || (space != RDR_HGRAD && !(hb[t] > 0))) return RDR_EINVAL;
  h->loop = loop;

  Mesh m;
  if ((st = build_mesh(hx.data(), nv, ht.data(), nt, hm.data(), m))) return st;
  const auto tr0 = std::chrono::steady_clock::now();
  const RefElement& el = reference_element(space, p);
  if (space == RDR_HCURL) reference_element(RDR_HGRAD, p);  // the potential space's, timed here too
  h->info.refelem_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - tr0).count();
  Numbering num;
  build_numbering(m, el, num);
  std::vector<double> coef;
  cell_coefficients(m, space, ha.data(), hb.data(), coef);
  h->space = space;
  h->p = p;
  h->n_total = num.n_total;

  // ---- operator
  EntityMap em;
  if (build_entity_map(m, num, el, em)) return RDR_EMESH;
  DevOperator& op = h->op;
  op.n_loc = el.n;
  op.n_mat = el.n_mat;
  op.n_cells = nt;
  op.n_total = num.n_total;
  uint16_t* d_lut;
  double *d_coef, *d_R;
  if ((st = h->own_upload(&d_lut, em.lut))) return st;
  if ((st = h->own_upload(&d_coef, coef))) return st;
  if ((st = h->own_upload(&d_R, el.R))) return st;  // the device patch setup's reference matrices
  op.lut = d_lut;
  op.coef = d_coef;
  op.R = d_R;
  op.kp = (el.n + 3) / 4 * 4;
  op.ngroups = (el.n + 31) / 32;
  {
    // The DMMA apply's local order. H(curl): the curl matrices R_6..R_11 (K^ab) are zero
    // on the gradient dofs (curl grad = 0; Eq. 3.14 splits every entity's Ned1 dofs into
    // gradients of H(grad) bubbles and the rest), up to rounding of the extended-precision
    // build (<= 1e-16 of max |K^ab|): those dofs go last, the ncb others first, and the
    // apply skips the curl matrices on chunks / column groups beyond ncb (kernels.cu).
    // H(div) likewise: the div-div matrix R_6 is zero on the divergence-free RT dofs
    // (curls of Ned1 bubbles, §3.4.3), 0.87 of the flops. Meshes below
    // kFactMinCells cells keep the element order and every entry (kernels.hpp).
    std::vector<int> perm(el.n);
    for (int i = 0; i < el.n; ++i) perm[i] = i;
    op.ncb = el.n;
    op.nm0 = space == RDR_HGRAD ? el.n_mat : 6;
    if (space != RDR_HGRAD && nt >= kFactMinCells) {  // H(div): R_6 likewise on the div-free dofs
      const size_t nn = (size_t)el.n * el.n;
      double mx = 0.0;
      for (int s = 6; s < el.n_mat; ++s)
        for (size_t k = 0; k < nn; ++k) mx = std::max(mx, std::fabs(el.R[s * nn + k]));
      std::vector<char> curl(el.n, 0);
      for (int s = 6; s < el.n_mat; ++s)
        for (int i = 0; i < el.n; ++i)
          for (int j = 0; j < el.n; ++j)
            if (std::fabs(el.R[s * nn + (size_t)i * el.n + j]) > 1e-12 * mx) curl[i] = curl[j] = 1;
      int k = 0;
      for (int i = 0; i < el.n; ++i)
        if (curl[i]) perm[k++] = i;
      op.ncb = k;
      for (int i = 0; i < el.n; ++i)
        if (!curl[i]) perm[k++] = i;
    }
    std::vector<uint16_t> lut_tc(el.n);
    for (int i = 0; i < el.n; ++i) lut_tc[i] = em.lut[perm[i]];
    uint16_t* d_lut_tc;
    if ((st = h->own_upload(&d_lut_tc, lut_tc))) return st;
    op.lut_tc = d_lut_tc;
    // reference matrices stacked j-major in 32-column groups: group g, chunk j4,
    // matrix s, row t holds R_s[4 j4 + t][32 g + c] (local order perm) at column
    // c ^ (t << 2) (the shared-memory swizzle of apply_tc_kernel's B fragments)
    const int nm = el.n_mat, nj4 = op.kp / 4;
    std::vector<double> B((size_t)op.ngroups * nj4 * nm * 4 * 32, 0.0);
    for (int g = 0; g < op.ngroups; ++g)
      for (int j4 = 0; j4 < nj4; ++j4)
        for (int s = 0; s < nm; ++s)
          for (int t = 0; t < 4; ++t) {
            const int j = 4 * j4 + t;
            if (j >= el.n) continue;
            const size_t row = (((size_t)g * nj4 + j4) * nm + s) * 4 + t;
            for (int c = 0; c < 32; ++c) {
              const int col = 32 * g + c;
              if (col < el.n && (s < 6 || (j < op.ncb && col < op.ncb)))
                B[row * 32 + (c ^ (t << 2))] = el.R[((size_t)s * el.n + perm[j]) * el.n + perm[col]];
            }
          }
    double* d_B;
    if ((st = h->own_upload(&d_B, B))) return st;
    op.Bsw = d_B;
  }
  op.F = nullptr;
  op.nf = op.nfm = op.nfp = op.fact = 0;
  op.fact_nsa = op.fact_nsb = 1;
  op.fck = space == RDR_HDIV ? 1 : 3;
  op.ubuf = nullptr;
  if (el.nf > 0) {  // factored apply: F [kp][nfp] zero-padded, stage-A buffer
    op.nf = el.nf;
    op.nfm = el.nfm;
    op.nfp = (el.nf + 31) / 32 * 32;
    std::vector<double> Fp((size_t)op.kp * op.nfp, 0.0);
    for (int i = 0; i < el.n; ++i)
      for (int j = 0; j < el.nf; ++j) Fp[(size_t)i * op.nfp + j] = el.F[(size_t)i * el.nf + j];
    double* d_F;
    if ((st = h->own_upload(&d_F, Fp))) return st;
    op.F = d_F;
    if ((st = h->own_alloc((void**)&op.ubuf, sizeof(double) * (size_t)nt * op.nfp))) return st;
  }
  if ((st = h->own_upload(&h->d_cons, num.constrained))) return st;
  {  // a layout that fits (n_loc too large for all: EINVAL); tuned below on the device
    int k = 0;
    while (k < apply_variant_count() && apply_configure_variant(op, k)) ++k;
    if (k == apply_variant_count()) return RDR_EINVAL;
  }

  // ---- preconditioner
  DevPrecond& pc = h->pc;
  pc.n_total = num.n_total;
  pc.out_scale = 1.0;
  pc.hybrid = 0;
  pc.s1 = pc.s2 = 1.0;
  pc.nc = 0;
  pc.off3 = num.off[3];
  std::vector<double> dinv;
  interior_inverse_diagonal(m, num, el, coef, dinv);
  if (unsplit) std::fill(dinv.begin(), dinv.end(), 0.0);  // no Jacobi: the patches contain the interiors
  double* d_dinv;
  if ((st = h->own_upload(&d_dinv, dinv))) return st;
  pc.dinv = d_dinv;
  Numbering cg_num;
  std::vector<double> cg_coef;
  const RefElement* cg_el = nullptr;
  if (space == RDR_HCURL) {
    cg_el = &reference_element(RDR_HGRAD, p);
    build_numbering(m, *cg_el, cg_num);
    // potential patches: A_V = G_V^T A G_V = CG stiffness weighted by beta (curl grad = 0)
    std::vector<double> zero(nt, 0.0);
    cell_coefficients(m, RDR_HGRAD, hb.data(), zero.data(), cg_coef);
    Gradient G;
    build_gradient(m, num, cg_num, G);
    pc.n_cg_iface = unsplit ? cg_num.n_total : cg_num.off[3];  // unsplit potential patches hold cell bubbles
    G.ptr.resize(pc.n_cg_iface + 1);
    G.col.resize(G.ptr.back());
    G.val.resize(G.ptr.back());
    int64_t* d_gp;
    int32_t* d_gc;
    double* d_gv;
    if ((st = h->own_upload(&d_gp, G.ptr))) return st;
    if ((st = h->own_upload(&d_gc, G.col))) return st;
    if ((st = h->own_upload(&d_gv, G.val))) return st;
    pc.g_ptr = d_gp;
    pc.g_col = d_gc;
    pc.g_val = d_gv;
  }
  Patches P;
  DeviceTiles sink;
  const auto tp0 = std::chrono::steady_clock::now();
  PatchAssembly pasm;
  const PatchLayout layout = kTileGroups;
  st = build_patches(m, num, el, coef, space == RDR_HCURL ? &cg_num : nullptr, cg_el,
                     space == RDR_HCURL ? &cg_coef : nullptr, P, sink, layout, unsplit, host_setup ? nullptr : &pasm);
  if (sink.d) h->owned.push_back(sink.d);
  if (st) return st;
  pc.n_patches = (int64_t)P.n.size();
  {  // mostly small patches (<= 4 tile rows, e.g. the H(curl) edge stars): 4-warp CTAs, 8 per SM.
    // Only small patches (H(div) edge stars): one per warp (patch_warp_kernel). Mixed sizes keep
    // one CTA per patch: a second launch for the small ones measured slower on configs 2, 4, 5
    // and 7 (profiles/round2/experiments/patch_launch_shape_ab.log, and round 1's 273 -> 320 us).
    int64_t small = 0;
    for (int32_t n : P.n) small += n <= 128;
    pc.ldg_warps = 2 * small > pc.n_patches ? 4 : 8;
    pc.n_big = small == pc.n_patches ? 0 : pc.n_patches;
  }
  pc.max_n = P.max_n;
  int32_t *d_pn, *d_idx;
  int64_t *d_io, *d_to;
  uint8_t* d_pk;
  if ((st = h->own_upload(&d_pn, P.n))) return st;
  if ((st = h->own_upload(&d_io, P.idx_off))) return st;
  if ((st = h->own_upload(&d_idx, P.idx))) return st;
  if ((st = h->own_upload(&d_to, P.tile_off))) return st;
  if ((st = h->own_upload(&d_pk, P.kind))) return st;
  pc.pn = d_pn;
  pc.idx_off = d_io;
  pc.idx = d_idx;
  pc.tile_off = d_to;
  pc.tiles = sink.d;
  pc.pkind = d_pk;
  if (!host_setup && pc.n_patches > 0) {  // patch matrices assembled and inverted on the GPU
    DevPatchSetup ds;
    ds.pn = d_pn;
    ds.pkind = d_pk;
    ds.tile_off = d_to;
    ds.tiles = sink.d;
    ds.layout = (int)layout;
    ds.R[0] = d_R;
    ds.coef[0] = d_coef;
    ds.nl[0] = el.n;
    ds.nm[0] = el.n_mat;
    if ((st = device_patch_setup(ds, P, pasm, cg_el, space == RDR_HCURL ? &cg_coef : nullptr,
                                 &h->info.patch_kernel_seconds)))
      return st;
  }
  h->info.patch_setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count();
  pc.npad_max = std::max(32, (P.max_n + 31) / 32 * 32);

  // ---- PCG workspace: one slab, the vectors every kernel of an iteration touches
  // first, then the operator's entity bases and owner bits, so that an L2
  // access-policy window can keep them resident while the patch kernel streams
  // the inverses through L2 (see the size rule below)
  const size_t vb = sizeof(double) * std::max<int64_t>(1, num.n_total);
  {
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t ebb = sizeof(int32_t) * em.ebase.size(), owb = sizeof(uint16_t) * em.own.size();
    const size_t slab_bytes = 7 * al(vb) + al(ebb) + al(owb);
    char* slab = nullptr;
    if ((st = h->own_alloc((void**)&slab, slab_bytes))) return st;
    size_t off = 0;
    for (double** v : {&h->d_z, &h->d_p, &h->d_p2, &h->d_q, &h->d_r, &h->d_x}) {
      *v = reinterpret_cast<double*>(slab + off);
      off += al(vb);
    }
    int32_t* eb = reinterpret_cast<int32_t*>(slab + off);
    off += al(ebb);
    uint16_t* ow = reinterpret_cast<uint16_t*>(slab + off);
    off += al(owb);
    h->d_b = reinterpret_cast<double*>(slab + off);
    CK(cudaMemcpy(eb, em.ebase.data(), ebb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ow, em.own.data(), owb, cudaMemcpyHostToDevice));
    op.ebase = eb;
    op.own = ow;
    const size_t hot = off;  // everything but b
    int dev = 0, max_win = 0, max_persist = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    h->l2_window = {};
    // Only when the whole hot region fits the persisting set-aside and is at most
    // 16 MB (1/8 of L2; config 2's is 7 MB: bench 10.84k vs 10.71k PCG it/s);
    // larger full windows measured within +-2 % (configs 4, 6) and a partial one
    // 4 % slower (config 3) (profiles/experiments/r2w_l2_persist_ab.log,
    // r2x_l2_persist_ab.log).
    const bool fits = hot <= (size_t)max_win && hot <= (size_t)max_persist;
    const bool want = hot <= ((size_t)16 << 20);
    if (fits && want) {
      const size_t bytes = hot, setaside = hot;
      l2_window_acquire(setaside);
      h->l2_window.base_ptr = slab;
      h->l2_window.num_bytes = bytes;
      h->l2_window.hitRatio = (float)setaside / (float)bytes;
      h->l2_window.hitProp = cudaAccessPropertyPersisting;
      h->l2_window.missProp = cudaAccessPropertyStreaming;
    }
    cudaGetLastError();  // the limit / attributes are hints: never fail the setup on them
  }
  h->fused = fused_pcg_supported(op) && !hybrid;
  if (hybrid) {  // ---- Whitney coarse space + sweep workspace + weights
    std::vector<int32_t> cidx;
    std::vector<double> ctiles, cdense;
    if ((st = build_coarse(m, num, el, coef, cidx, ctiles, host_setup ? nullptr : &cdense))) return st;
    pc.nc = (int64_t)cidx.size();
    int32_t* d_cidx;
    double* d_ct = nullptr;
    if ((st = h->own_upload(&d_cidx, cidx))) return st;
    if (host_setup) {
      if ((st = h->own_upload(&d_ct, ctiles))) return st;
    } else if (pc.nc > 0) {  // device inverse of the coarse matrix (multi-CTA block sweep)
      const int nc = (int)pc.nc;
      const int64_t ld = (nc + 63) / 64 * 64;
      if ((st = h->own_alloc((void**)&d_ct, sizeof(double) * patch_stored_doubles(nc)))) return st;
      CK(cudaMemset(d_ct, 0, sizeof(double) * patch_stored_doubles(nc)));
      DevTemps tmp;
      double *dA = nullptr, *work = nullptr;
      int32_t* dst = nullptr;
      CK(cudaMalloc((void**)&dA, sizeof(double) * ld * ld));
      tmp.p.push_back(dA);
      CK(cudaMalloc((void**)&work, sizeof(double) * (64 * 64 + 2 * 64 * ld)));
      tmp.p.push_back(work);
      CK(cudaMalloc((void**)&dst, sizeof(int32_t)));
      tmp.p.push_back(dst);
      CK(cudaMemset(dst, 0, sizeof(int32_t)));
      CK(cudaMemset(dA, 0, sizeof(double) * ld * ld));
      CK(cudaMemcpy2D(dA, sizeof(double) * ld, cdense.data(), sizeof(double) * nc, sizeof(double) * nc, nc,
                      cudaMemcpyHostToDevice));
      CK(dense_spd_inverse_packed(dA, ld, nc, work, dst, d_ct, (int)kTileGroups, 0));
      int32_t bad = 0;
      CK(cudaMemcpy(&bad, dst, sizeof(int32_t), cudaMemcpyDeviceToHost));
      if (bad) return RDR_ENOTSPD;
    }
    pc.cidx = d_cidx;
    pc.ctiles = d_ct;
    if ((st = h->own_alloc((void**)&pc.czc, sizeof(double) * std::max<int64_t>(1, pc.nc)))) return st;
    if ((st = h->own_alloc((void**)&pc.ht, vb))) return st;
    if ((st = h->own_alloc((void**)&pc.hy, vb))) return st;
    if ((st = hybrid_weights(h, dinv))) return st;
    pc.hybrid = 1;
  }
  if ((st = h->own_alloc((void**)&h->d_sc, sizeof(PcgScalars)))) return st;
  CK(cudaMallocHost((void**)&h->h_sc, sizeof(PcgScalars)));
  CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  if (h->l2_window.num_bytes) {  // captured into the kernel nodes of the solve graphs
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow = h->l2_window;
    if (cudaStreamSetAttribute(h->cap_stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess)
      cudaGetLastError();
  }
  h->launches_per_iter = h->fused ? 1 + count_precond_launches(pc)
                                  : 4 + (hybrid ? count_hybrid_launches(pc) : count_precond_launches(pc));
  // one warm-up apply/precond on zero vectors: kernel attributes get configured
  // here, outside any later stream capture
  CK(cudaMemset(h->d_p, 0, vb));
  {  // the fastest warp layout on this operator, timed on the PCG-mode apply with x = 1 (the
     // scalars: rtol 0, huge maxit -- the stopping test never fires)
    std::vector<double> ones(num.n_total, 1.0);
    CK(cudaMemcpy(h->d_b, ones.data(), vb, cudaMemcpyHostToDevice));
    std::memset(h->h_sc, 0, sizeof(PcgScalars));
    h->h_sc->maxit = 1 << 30;
    CK(cudaMemcpy(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice));
    if (tune_apply(op, h->d_b, h->d_q, h->d_sc, h->d_p, h->d_p2, 0, 5)) return RDR_ECUDA;
    if (tune_fact(op, pc, h->d_b, h->d_cons, h->d_x, h->d_r, h->d_z, h->d_q, h->d_sc, h->h_sc, h->d_p, h->d_p2, 0, 5))
      return RDR_ECUDA;
    if (op.fact && h->fused) h->launches_per_iter += 1;  // two stage kernels instead of one apply
    CK(cudaMemset(h->d_p, 0, vb));
    CK(cudaMemset(h->d_p2, 0, vb));
  }
  if (tune_small_patches(pc, h->d_p, h->d_z, 0, 3)) return RDR_ECUDA;
  CK(launch_apply(op, h->d_p, h->d_q, nullptr, nullptr, 0));
  if (hybrid)
    CK(launch_precond_hybrid(op, pc, h->d_p, h->d_z, nullptr, 0));
  else
    CK(launch_precond(pc, h->d_p, h->d_z, nullptr, nullptr, 0));

  // ---- info
  rdr_info& in = h->info;
  in.n_total = num.n_total;
  int64_t nfree = 0;
  for (uint8_t c : num.constrained) nfree += !c;
  in.n_free = nfree;
  in.n_interior = num.n_total - num.off[3];
  in.n_cells = nt;
  in.n_loc = el.n;
  in.n_mat = el.n_mat;
  in.n_patches = pc.n_patches;
  in.max_patch = P.max_n;
  in.patch_bytes = P.total_doubles * 8;
  in.flops_apply = 2.0 * el.n * (double)el.n * el.n_mat * (double)nt;
  in.bytes_apply = 24.0 * num.n_total + (double)nt * (4.0 * el.n + 8.0 * el.n_mat);
  in.bytes_precond = P.alg_bytes + 24.0 * in.n_interior;
  in.persistent_loop = 0;
  in.apply_variant = op.av;
  in.apply_grid = op.apply_grid;
  in.apply_slots = op.apply_slots;
  in.small_patch_grid = pc.small_grid;
  in.apply_factored = op.fact;
  in.apply_fact_split_a = op.fact ? op.fact_nsa : 0;
  in.apply_fact_split_b = op.fact ? op.fact_nsb : 0;
  in.patch_setup_flops = 0;
  for (int32_t n : P.n) {  // lower tiles I >= J, I, J != K: nb(nb-1)/2 per K; panel: nb-1 per K
    const double nb = (n + 63) / 64;
    in.patch_setup_flops += 2.0 * 64 * 64 * 64 * nb * ((nb - 1) * nb / 2 + (nb - 1));
  }
  CK(cudaDeviceSynchronize());
  in.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return RDR_OK;
}

// rho_m = (lambda_min + 3 lambda_max) / 4 of a~_m^-1 A on X_m from 10 CG
// (Lanczos) steps with the splitmix64 rhs restricted to X_m (
// oracle/hybrid.py does the same on the CPU): X_1 = interior dofs with the
// point-Jacobi solver, X_2 = free interface dofs with the additive patches.
static int hybrid_weights(rdr_handle* h, const std::vector<double>& dinv) {
  const int64_t n = h->n_total, off3 = h->pc.off3;
  std::vector<uint8_t> cons(n);
  CK(cudaMemcpy(cons.data(), h->d_cons, n, cudaMemcpyDeviceToHost));
  const size_t vb = sizeof(double) * n;
  for (int m = 0; m < 2; ++m) {
    std::vector<double> mask(n, 0.0);
    int64_t dim = 0;
    for (int64_t i = 0; i < n; ++i)
      if (m == 0 ? i >= off3 : (i < off3 && !cons[i])) {
        mask[i] = 1.0;
        ++dim;
      }
    if (dim == 0) {
      (m == 0 ? h->pc.s1 : h->pc.s2) = 1.0;
      continue;
    }
    std::vector<double> r(n), z(n), pv(n), q(n);
    auto applyA = [&](const std::vector<double>& v, std::vector<double>& out) -> int {
      CK(cudaMemcpy(h->d_p, v.data(), vb, cudaMemcpyHostToDevice));
      CK(cudaMemset(h->d_q, 0, vb));
      CK(launch_apply(h->op, h->d_p, h->d_q, nullptr, nullptr, 0));
      CK(cudaMemcpy(out.data(), h->d_q, vb, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i) out[i] *= mask[i];
      return RDR_OK;
    };
    auto applyP = [&](const std::vector<double>& v, std::vector<double>& out) -> int {
      if (m == 0) {
        for (int64_t i = 0; i < n; ++i) out[i] = i >= off3 ? dinv[i - off3] * v[i] : 0.0;
        return RDR_OK;
      }
      CK(cudaMemcpy(h->d_r, v.data(), vb, cudaMemcpyHostToDevice));
      CK(cudaMemset(h->d_z, 0, vb));
      CK(launch_precond_part(1, h->pc, h->d_r, h->d_z, nullptr, nullptr, 0));
      CK(cudaMemcpy(out.data(), h->d_z, vb, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i) out[i] *= mask[i];
      return RDR_OK;
    };
    auto dot = [&](const std::vector<double>& a, const std::vector<double>& b) {
      double s = 0;
      for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
      return s;
    };
    int st;
    for (int64_t i = 0; i < n; ++i) r[i] = mask[i] * splitmix_uniform(kLanczosSeed, (uint64_t)i);
    if ((st = applyP(r, z))) return st;
    pv = z;
    double rz = dot(r, z);
    std::vector<double> alphas, betas;
    for (int k = 0; k < kLanczosSteps && rz > 0; ++k) {
      if ((st = applyA(pv, q))) return st;
      const double a = rz / dot(pv, q);
      alphas.push_back(a);
      for (int64_t i = 0; i < n; ++i) r[i] -= a * q[i];
      if ((st = applyP(r, z))) return st;
      const double rz_new = dot(r, z), beta = rz_new / rz;
      betas.push_back(beta);
      for (int64_t i = 0; i < n; ++i) pv[i] = z[i] + beta * pv[i];
      rz = rz_new;
    }
    const int k = (int)alphas.size();
    std::vector<double> T((size_t)k * k, 0.0);
    for (int j = 0; j < k; ++j) {
      T[j * k + j] = 1.0 / alphas[j] + (j > 0 ? betas[j - 1] / alphas[j - 1] : 0.0);
      if (j + 1 < k) T[j * k + j + 1] = T[(j + 1) * k + j] = std::sqrt(betas[j]) / alphas[j];
    }
    const std::vector<double> ev = sym_eigenvalues(T, k);
    const double rho = k > 0 ? (ev.front() + 3.0 * ev.back()) / 4.0 : 1.0;
    (m == 0 ? h->pc.s1 : h->pc.s2) = 1.0 / rho;
    (m == 0 ? h->rho1 : h->rho2) = rho;
  }
  return RDR_OK;
}

extern "C" {

int rdr_setup_ex(rdr_handle** hp, const double* vertices, int64_t nv, const int32_t* tets, int64_t nt, int p,
                 int space, const double* alpha, const double* beta, const uint8_t* dirichlet_mask,
                 const rdr_options* opt, void* stream) {
  if (!hp) return RDR_EINVAL;
  *hp = nullptr;
  if (!vertices || !tets || !alpha || !beta || !dirichlet_mask || nv < 4 || nt < 1) return RDR_EINVAL;
  if (space != RDR_HGRAD && space != RDR_HCURL && space != RDR_HDIV) return RDR_EINVAL;
  if (p < 1 || (space == RDR_HGRAD && p > 12) || (space != RDR_HGRAD && p > 10)) return RDR_EINVAL;
  if (nv > 0x7fffffff || nt > 0x7fffffff) return RDR_EINVAL;
  const int dec = opt ? opt->decomposition : RDR_SPLIT;
  if (dec != RDR_SPLIT && dec != RDR_UNSPLIT) return RDR_EINVAL;
  const int pre = opt ? opt->preconditioner : RDR_ADDITIVE;
  if (pre != RDR_ADDITIVE && pre != RDR_HYBRID) return RDR_EINVAL;
  if (pre == RDR_HYBRID && dec != RDR_SPLIT) return RDR_EINVAL;
  const int su = opt ? opt->setup : RDR_SETUP_DEVICE;
  if (su != RDR_SETUP_DEVICE && su != RDR_SETUP_HOST) return RDR_EINVAL;
  const int loop = opt ? opt->loop : RDR_LOOP_DEVICE;
  if (loop < RDR_LOOP_DEVICE || loop > RDR_LOOP_PERSISTENT) return RDR_EINVAL;
  rdr_handle* h = new (std::nothrow) rdr_handle();
  if (!h) return RDR_ENOMEM;
  int st;
  try {
    st = setup_impl(h, vertices, nv, tets, nt, p, space, alpha, beta, dirichlet_mask, dec == RDR_UNSPLIT,
                    pre == RDR_HYBRID, su == RDR_SETUP_HOST, loop, (cudaStream_t)stream);
  } catch (const std::bad_alloc&) {
    st = RDR_ENOMEM;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rdr_setup: %s\n", e.what());
    st = RDR_EINVAL;
  }
  if (!st) st = select_loop(h);
  if (st) {
    delete h;
    return st;
  }
  *hp = h;
  return RDR_OK;
}

int rdr_setup(rdr_handle** hp, const double* vertices, int64_t nv, const int32_t* tets, int64_t nt, int p, int space,
              const double* alpha, const double* beta, const uint8_t* dirichlet_mask, void* stream) {
  return rdr_setup_ex(hp, vertices, nv, tets, nt, p, space, alpha, beta, dirichlet_mask, nullptr, stream);
}

int rdr_ndofs(const rdr_handle* h, int64_t* n_total) {
  if (!h || !n_total) return RDR_EINVAL;
  *n_total = h->n_total;
  return RDR_OK;
}

int rdr_get_info(const rdr_handle* h, rdr_info* out) {
  if (!h || !out) return RDR_EINVAL;
  *out = h->info;
  return RDR_OK;
}

int rdr_apply(rdr_handle* h, const double* x, double* y, void* stream) {
  if (!h || !x || !y) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemsetAsync(y, 0, sizeof(double) * h->n_total, s));
  CK(launch_apply(h->op, x, y, nullptr, nullptr, s));
  return RDR_OK;
}

int rdr_precond(rdr_handle* h, const double* r, double* z, void* stream) {
  if (!h || !r || !z) return RDR_EINVAL;
  if (h->pc.hybrid)
    CK(launch_precond_hybrid(h->op, h->pc, r, z, nullptr, (cudaStream_t)stream));
  else
    CK(launch_precond(h->pc, r, z, nullptr, nullptr, (cudaStream_t)stream));
  return RDR_OK;
}

int rdr_get_weights(const rdr_handle* h, double* rho) {
  if (!h || !rho) return RDR_EINVAL;
  rho[0] = h->rho1;
  rho[1] = h->rho2;
  rho[2] = 1.0;
  return RDR_OK;
}

static int enqueue_iteration(rdr_handle* h, cudaStream_t s) {
  const int64_t n = h->n_total;
  if (h->fused) {  // 3 kernels per PCG iteration
    CK(launch_pcg_fused_apply(h->op, h->d_sc, h->d_z, h->d_p, h->d_p2, h->d_q, s));
    CK(launch_pcg_update_jacobi(h->d_sc, h->pc, h->d_p, h->d_p2, h->d_q, h->d_x, h->d_r, h->d_z, s));
    CK(launch_precond_part(1, h->pc, h->d_r, h->d_z, &h->d_sc->rz_acc, h->d_sc, s));
    return RDR_OK;
  }
  CK(launch_apply(h->op, h->d_p, h->d_q, &h->d_sc->pq, h->d_sc, s));
  CK(launch_pcg_update(h->d_sc, h->d_p, h->d_q, h->d_x, h->d_r, n, s));
  if (h->pc.hybrid) {  // r.z of the new z in the finish kernel's pass over z
    CK(launch_precond_hybrid(h->op, h->pc, h->d_r, h->d_z, h->d_sc, s));
  } else {
    CK(launch_precond(h->pc, h->d_r, h->d_z, &h->d_sc->rz_new, h->d_sc, s));
  }
  CK(launch_pcg_finish(h->d_sc, h->d_z, h->pc.hybrid ? h->d_r : nullptr, n, s));
  CK(launch_pcg_direction(h->d_sc, h->d_z, h->d_p, h->d_q, n, s));
  return RDR_OK;
}

static int build_graph(rdr_handle* h, int iters) {
  if (h->graph) return RDR_OK;
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  int st = RDR_OK;
  for (int k = 0; k < iters && st == RDR_OK; ++k) st = enqueue_iteration(h, h->cap_stream);
  cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
  if (st) return st;
  CK(e);
  e = cudaGraphInstantiate(&h->graph, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  h->graph_iters = iters;
  return RDR_OK;
}

// Device-side PCG loop: one graph whose while node repeats a body of
// while_unroll(h) iterations until the stopping test (inside the fused apply;
// pcg_finish_kernel on the unfused path) clears the condition, so a whole
// solve is one graph launch and one host synchronisation. (Fused path: a body
// per iteration measured ~3 us/iteration slower than the host-driven
// 8-iteration graphs: the conditional node's body launch is not free, so it is
// amortised over several iterations. The hybrid sweep is 20+ launches per
// iteration and converges in 10-25 iterations, so its body is one iteration:
// nothing runs past the iteration that converged.)
constexpr int kWhileUnroll = 8;
static int while_unroll(const rdr_handle* h) { return h->fused ? kWhileUnroll : h->pc.hybrid ? 1 : 4; }
static int build_while_graph(rdr_handle* h) {
  if (h->wgraph) return RDR_OK;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle loop;
  CK(cudaGraphConditionalHandleCreate(&loop, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams params = {};
  params.type = cudaGraphNodeTypeConditional;
  params.conditional.handle = loop;
  params.conditional.type = cudaGraphCondTypeWhile;
  params.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &params));
  cudaGraph_t body = params.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(h->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int st = RDR_OK;
  for (int k = 0; k < while_unroll(h) && st == RDR_OK; ++k) st = enqueue_iteration(h, h->cap_stream);
  if (st == RDR_OK) {
    cudaError_t ce = launch_pcg_loop_condition(h->d_sc, loop, h->cap_stream);
    if (ce != cudaSuccess) st = cuda_status(ce);
  }
  cudaError_t e = cudaStreamEndCapture(h->cap_stream, &body);
  if (st) return st;
  CK(e);
  e = cudaGraphInstantiate(&h->wgraph, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  return RDR_OK;
}

// PCG start (R-A16): x0 = 0, r0 = b (masked), z0 = P^-1 r0 and the scalars;
// returns the launches it enqueued
static int64_t pcg_begin(rdr_handle* h, const double* b, double rtol, int maxit, cudaStream_t s, int* st) {
  const int64_t n = h->n_total;
  auto fail = [&](cudaError_t e) {
    *st = cuda_status(e);
    return (int64_t)0;
  };
  cudaError_t e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e);  // h_sc (pinned) is the H2D template
  std::memset(h->h_sc, 0, sizeof(PcgScalars));
  if (h->fused) {
    h->h_sc->rtol = rtol;
    h->h_sc->maxit = maxit;
    if ((e = cudaMemcpyAsync(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice, s))) return fail(e);
    if ((e = cudaMemsetAsync(h->d_p, 0, sizeof(double) * n, s))) return fail(e);
    if ((e = cudaMemsetAsync(h->d_p2, 0, sizeof(double) * n, s))) return fail(e);
    if ((e = launch_pcg_init(b, h->d_cons, n, h->d_x, h->d_r, h->d_q, s))) return fail(e);
    if ((e = launch_precond(h->pc, h->d_r, h->d_z, &h->d_sc->rz_acc, nullptr, s))) return fail(e);
    *st = RDR_OK;
    return 1 + count_precond_launches(h->pc);
  }
  if ((e = cudaMemcpyAsync(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice, s))) return fail(e);
  if ((e = launch_pcg_init(b, h->d_cons, n, h->d_x, h->d_r, h->d_q, s))) return fail(e);
  if (h->pc.hybrid) {
    if ((e = launch_precond_hybrid(h->op, h->pc, h->d_r, h->d_z, nullptr, s))) return fail(e);
    if ((e = launch_pcg_rz(h->d_sc, h->d_r, h->d_z, n, s))) return fail(e);
  } else {
    if ((e = launch_precond(h->pc, h->d_r, h->d_z, &h->d_sc->rz_new, nullptr, s))) return fail(e);
  }
  if ((e = launch_pcg_start(h->d_sc, h->d_z, h->d_p, n, rtol, maxit, s))) return fail(e);
  *st = RDR_OK;
  return 2 + (h->pc.hybrid ? count_hybrid_launches(h->pc) + 1 : count_precond_launches(h->pc));
}

static int fetch_scalars(rdr_handle* h, cudaStream_t s) {
  CK(cudaMemcpyAsync(h->h_sc, h->d_sc, sizeof(PcgScalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return RDR_OK;
}

// One PCG solve. rdr_options.loop: RDR_LOOP_DEVICE -- one graph whose while node
// repeats 8-iteration bodies until the device-side stopping test fires (one host
// synchronisation per solve; the hybrid preconditioner's unfused iteration with a
// one-iteration body); RDR_LOOP_HOST -- graphs of 8 iterations relaunched by the host
// until done; RDR_LOOP_EAGER -- every kernel launched on the stream, the host
// checking the stop flag after each iteration (no graphs: profilers see every
// launch).
static int solve_device(rdr_handle* h, const double* b, double rtol, int maxit, int* iters, cudaStream_t s) {
  int st;
  if (h->use_persist) {  // the whole solve in one cooperative launch (small problems)
    CK(cudaStreamSynchronize(s));
    std::memset(h->h_sc, 0, sizeof(PcgScalars));
    h->h_sc->rtol = rtol;
    h->h_sc->maxit = maxit;
    CK(cudaMemcpyAsync(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice, s));
    CK(launch_persistent_pcg(h->persist, h->op, h->pc, h->d_sc, b, h->d_cons, h->d_x, h->d_r, h->d_z, h->d_p,
                             h->d_p2, h->d_q, s));
    if ((st = fetch_scalars(h, s))) return st;
    h->last_launches = 1;
    *iters = h->h_sc->iters;
    return h->h_sc->converged ? RDR_OK : RDR_ENOCONV;
  }
  int64_t launches = pcg_begin(h, b, rtol, maxit, s, &st);
  if (st) return st;
  // the unfused path tests before each iteration, the fused one inside its apply
  const bool test_first = !h->fused;
  if (h->loop == RDR_LOOP_DEVICE || h->loop == RDR_LOOP_GRAPH) {
    if ((st = build_while_graph(h))) return st;
    CK(cudaGraphLaunch(h->wgraph, s));
    if ((st = fetch_scalars(h, s))) return st;
    // bodies of U iterations (+ the condition kernel) ran until the one that detected convergence
    // (fused: k counts the fused applies; unfused: the first body always runs, its kernels
    // returning at once when the start already set the stop flag)
    const int U = while_unroll(h);
    const int64_t steps = h->fused ? h->h_sc->k : std::max(h->h_sc->iters, 1);
    const int64_t bodies = (steps + U - 1) / U;
    launches += bodies * ((int64_t)U * h->launches_per_iter + 1);
  } else if (h->loop == RDR_LOOP_EAGER) {
    for (;;) {
      if (test_first) {
        if ((st = fetch_scalars(h, s))) return st;
        if (h->h_sc->done) break;
      }
      if ((st = enqueue_iteration(h, s))) return st;
      launches += h->launches_per_iter;
      if (!test_first) {
        if ((st = fetch_scalars(h, s))) return st;
        if (h->h_sc->done) break;
      }
    }
  } else {
    if ((st = build_graph(h, 8))) return st;
    for (;;) {
      if (test_first) {
        if ((st = fetch_scalars(h, s))) return st;
        if (h->h_sc->done) break;
      }
      CK(cudaGraphLaunch(h->graph, s));
      launches += (int64_t)h->graph_iters * h->launches_per_iter;
      if (!test_first) {
        if ((st = fetch_scalars(h, s))) return st;
        if (h->h_sc->done) break;
      }
    }
  }
  h->last_launches = launches;
  *iters = h->h_sc->iters;
  return h->h_sc->converged ? RDR_OK : RDR_ENOCONV;
}

}  // extern "C"

// rdr_options.loop: RDR_LOOP_DEVICE runs a small problem's solves as one
// persistent cooperative launch when the kernel is eligible (additive
// preconditioner, patches <= 256 dofs, n_loc <= 128, its shared memory fits) and
// a 40-iteration solve measured at setup is faster than with the graph's WHILE
// node; RDR_LOOP_PERSISTENT requires it (RDR_EINVAL if not eligible);
// RDR_LOOP_GRAPH, RDR_LOOP_HOST and RDR_LOOP_EAGER never use it.
static int select_loop(rdr_handle* h) {
  h->use_persist = false;
  if (!h->fused || (h->loop != RDR_LOOP_DEVICE && h->loop != RDR_LOOP_PERSISTENT)) return RDR_OK;
  h->persist = plan_persistent_pcg(h->op, h->pc);
  if (h->persist.grid == 0) return h->loop == RDR_LOOP_PERSISTENT ? RDR_EINVAL : RDR_OK;
  if (h->loop == RDR_LOOP_PERSISTENT) {
    h->use_persist = true;
    h->info.persistent_loop = 1;
    return RDR_OK;
  }
  // time both drivers on a 40-iteration solve (rtol 0; a typical length) with b = 1 on every dof
  std::vector<double> ones(h->n_total, 1.0);
  CK(cudaMemcpy(h->d_b, ones.data(), sizeof(double) * h->n_total, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float t[2] = {0.f, 0.f};
  for (int mode = 0; mode < 2; ++mode) {
    h->use_persist = mode == 1;
    int it = 0, st = RDR_OK;
    for (int rep = 0; rep < 3 && (st == RDR_OK || st == RDR_ENOCONV); ++rep) {  // the last one timed
      CK(cudaEventRecord(e0, 0));
      st = solve_device(h, h->d_b, 0.0, 40, &it, 0);
      CK(cudaEventRecord(e1, 0));
      CK(cudaEventSynchronize(e1));
    }
    if (st != RDR_OK && st != RDR_ENOCONV) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return st;
    }
    CK(cudaEventElapsedTime(&t[mode], e0, e1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  h->use_persist = t[1] < t[0];
  h->info.persistent_loop = h->use_persist;
  return RDR_OK;
}

extern "C" {

int rdr_solve(rdr_handle* h, const double* b, double* x, double rtol, int maxit, int* iters, void* stream) {
  if (!h || !b || !x || !iters || !(rtol >= 0)) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  int st = solve_device(h, b, rtol, maxit, iters, s);
  if (st != RDR_OK && st != RDR_ENOCONV) return st;
  CK(cudaMemcpyAsync(x, h->d_x, sizeof(double) * h->n_total, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  return st;
}

int rdr_solve_host(rdr_handle* h, const double* b_host, double* x_host, double rtol, int maxit, int* iters,
                   void* stream) {
  if (!h || !b_host || !x_host || !iters || !(rtol >= 0)) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(h->d_b, b_host, sizeof(double) * h->n_total, cudaMemcpyHostToDevice, s));
  int st = solve_device(h, h->d_b, rtol, maxit, iters, s);
  if (st != RDR_OK && st != RDR_ENOCONV) return st;
  CK(cudaMemcpyAsync(x_host, h->d_x, sizeof(double) * h->n_total, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return st;
}

int rdr_debug_fused_apply(rdr_handle* h, const double* z, double* q, void* stream) {
  // one fused PCG apply at iteration 0 (p_0 = z): q = A z, for debugging the PCG mode of the kernel
  if (!h || !z || !q || !h->fused) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = h->n_total;
  CK(cudaStreamSynchronize(s));
  std::memset(h->h_sc, 0, sizeof(PcgScalars));
  h->h_sc->rtol = 0.0;
  h->h_sc->maxit = 1000;
  CK(cudaMemcpyAsync(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(h->d_p, 0, sizeof(double) * n, s));
  CK(cudaMemsetAsync(h->d_p2, 0, sizeof(double) * n, s));
  CK(cudaMemsetAsync(q, 0, sizeof(double) * n, s));
  CK(launch_pcg_fused_apply(h->op, h->d_sc, z, h->d_p, h->d_p2, q, s));
  CK(cudaStreamSynchronize(s));
  return RDR_OK;
}

int rdr_debug_set_apply_variant(rdr_handle* h, int variant) {
  if (!h) return RDR_EINVAL;
  DevOperator t = h->op;
  if (apply_configure_variant(t, variant)) return RDR_EINVAL;
  if (t.fact && h->fused) h->launches_per_iter -= 1;
  t.fact = 0;
  h->info.apply_factored = 0;
  h->info.apply_fact_split_a = h->info.apply_fact_split_b = 0;
  h->op = t;
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->wgraph) cudaGraphExecDestroy(h->wgraph);
  h->graph = h->wgraph = nullptr;  // captured with the old launch configuration
  h->info.apply_variant = t.av;
  h->info.apply_grid = t.apply_grid;
  h->info.apply_slots = t.apply_slots;
  return RDR_OK;
}

int rdr_debug_set_apply_config(rdr_handle* h, int variant, int slots, int grid) {
  if (!h) return RDR_EINVAL;
  DevOperator t = h->op;
  if (variant <= -1 && variant >= -3) {  // the factored two-stage apply, tile sizes op.fact = -variant
    const int f = -variant;
    if (!fact_apply_fits(t, f)) return RDR_EINVAL;
    if (slots < 0 || slots > 8 || grid < 0 || grid > 8) return RDR_EINVAL;
    if (!t.fact && h->fused) h->launches_per_iter += 1;
    t.fact = f;
    t.fact_nsa = std::max(1, slots);  // factored: slots / grid carry the column splits of stage A / B
    t.fact_nsb = std::max(1, grid);
  } else {
    if (apply_configure_exact(t, variant, slots, grid)) return RDR_EINVAL;
    if (t.fact && h->fused) h->launches_per_iter -= 1;
    t.fact = 0;
  }
  h->info.apply_factored = t.fact;
  h->info.apply_fact_split_a = t.fact ? t.fact_nsa : 0;
  h->info.apply_fact_split_b = t.fact ? t.fact_nsb : 0;
  h->op = t;
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->wgraph) cudaGraphExecDestroy(h->wgraph);
  h->graph = h->wgraph = nullptr;  // captured with the old launch configuration
  h->info.apply_variant = t.av;
  h->info.apply_grid = t.apply_grid;
  h->info.apply_slots = t.apply_slots;
  return RDR_OK;
}

int rdr_debug_set_small_patch_kernel(rdr_handle* h, int persistent) {
  if (!h || h->pc.n_big >= h->pc.n_patches || (persistent != 0 && persistent != 1)) return RDR_EINVAL;
  if (!persistent) {
    h->pc.small_grid = 0;
  } else {
    DevPrecond t = h->pc;
    // reuse the tuner's occupancy-based grid: time nothing, take the persistent grid
    const int W = t.ldg_warps;
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t needed = (t.n_patches - t.n_big + W - 1) / W;
    h->pc.small_grid = (int)std::min<int64_t>(needed, (int64_t)sms * (24 / W));
  }
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->wgraph) cudaGraphExecDestroy(h->wgraph);
  h->graph = h->wgraph = nullptr;  // captured with the old launch configuration
  h->info.small_patch_grid = h->pc.small_grid;
  return RDR_OK;
}

int rdr_last_launches(const rdr_handle* h, int64_t* launches) {
  if (!h || !launches) return RDR_EINVAL;
  *launches = h->last_launches;
  return RDR_OK;
}

int rdr_last_solve(const rdr_handle* h, rdr_solve_stats* out) {
  if (!h || !out) return RDR_EINVAL;
  out->iters = h->h_sc->iters;
  out->converged = h->h_sc->converged;
  out->z0 = h->h_sc->z0;
  out->z_last = h->h_sc->z_last;
  out->launches = h->last_launches;
  return RDR_OK;
}

int rdr_profile_solve(rdr_handle* h, const double* b, double rtol, int maxit, int* iters, double* ms, void* stream) {
  if (!h || !b || !iters || !ms || !(rtol >= 0)) return RDR_EINVAL;
  if (!h->fused) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  int st;
  pcg_begin(h, b, rtol, maxit, s, &st);
  if (st) return st;
  cudaEvent_t ev[4];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[4] = {0, 0, 0, 0};
  int n_apply = 0;
  for (;;) {  // the eager fused iteration with an event between its kernel groups
    CK(cudaEventRecord(ev[0], s));
    CK(launch_pcg_fused_apply(h->op, h->d_sc, h->d_z, h->d_p, h->d_p2, h->d_q, s));
    CK(cudaEventRecord(ev[1], s));
    CK(launch_pcg_update_jacobi(h->d_sc, h->pc, h->d_p, h->d_p2, h->d_q, h->d_x, h->d_r, h->d_z, s));
    CK(cudaEventRecord(ev[2], s));
    CK(launch_precond_part(1, h->pc, h->d_r, h->d_z, &h->d_sc->rz_acc, h->d_sc, s));
    CK(cudaEventRecord(ev[3], s));
    if ((st = fetch_scalars(h, s))) break;
    float t[3];
    for (int k = 0; k < 3; ++k) CK(cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]));
    ++n_apply;
    if (h->h_sc->done) {  // this iteration's apply performed the final stopping test
      acc[0] += t[0];
      break;
    }
    acc[0] += t[0];
    acc[1] += t[1];
    acc[2] += t[2];
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (st) return st;
  const int n_full = std::max(1, n_apply - 1);
  ms[0] = acc[0] / n_apply;
  ms[1] = acc[1] / n_full;
  ms[2] = acc[2] / n_full;
  ms[3] = acc[3] / n_full;
  *iters = h->h_sc->iters;
  return h->h_sc->converged ? RDR_OK : RDR_ENOCONV;
}

// body of rdr_debug_profile_clocks (the caller owns d_acc and the events)
static int profile_clocks(rdr_handle* h, const double* b, int iters, double* out, cudaStream_t s, double* d_acc,
                          cudaEvent_t e0, cudaEvent_t e1) {
  constexpr unsigned kProbeNs = 10000;
  CK(cudaMemsetAsync(d_acc, 0, 4 * sizeof(double), s));
  float t[2] = {0.f, 0.f};
  for (int mode = 0; mode < 2; ++mode) {
    // mode 0: the PCG iteration (rtol 0: `iters` + 2 iterations whatever the residual), a probe
    // behind each fused apply; mode 1: the fused apply alone, back to back, a probe behind each
    int st;
    pcg_begin(h, b, 0.0, 1 << 30, s, &st);
    if (st) return st;
    auto step = [&]() -> int {
      CK(launch_pcg_fused_apply(h->op, h->d_sc, h->d_z, h->d_p, h->d_p2, h->d_q, s));
      CK(launch_sm_clock_probe(d_acc + 2 * mode, kProbeNs, s));
      if (mode == 0) {
        CK(launch_pcg_update_jacobi(h->d_sc, h->pc, h->d_p, h->d_p2, h->d_q, h->d_x, h->d_r, h->d_z, s));
        CK(launch_precond_part(1, h->pc, h->d_r, h->d_z, &h->d_sc->rz_acc, h->d_sc, s));
      }
      return RDR_OK;
    };
    for (int k = 0; k < 2; ++k)  // warm-up
      if ((st = step())) return st;
    CK(cudaMemsetAsync(d_acc + 2 * mode, 0, 2 * sizeof(double), s));
    CK(cudaEventRecord(e0, s));
    for (int k = 0; k < iters; ++k)
      if ((st = step())) return st;
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&t[mode], e0, e1));
  }
  double acc[4] = {0, 0, 0, 0};
  CK(cudaMemcpy(acc, d_acc, sizeof(acc), cudaMemcpyDeviceToHost));
  out[0] = acc[1] > 0 ? acc[0] / acc[1] : 0.0;
  out[1] = acc[3] > 0 ? acc[2] / acc[3] : 0.0;
  out[2] = t[0] / iters - kProbeNs * 1e-6;
  out[3] = t[1] / iters - kProbeNs * 1e-6;
  return RDR_OK;
}

int rdr_debug_profile_clocks(rdr_handle* h, const double* b, int iters, double* out, void* stream) {
  if (!h || !b || !out || iters < 1 || !h->fused) return RDR_EINVAL;
  double* d_acc = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int st = RDR_ECUDA;
  if (cudaMalloc((void**)&d_acc, 4 * sizeof(double)) == cudaSuccess && cudaEventCreate(&e0) == cudaSuccess &&
      cudaEventCreate(&e1) == cudaSuccess)
    st = profile_clocks(h, b, iters, out, (cudaStream_t)stream, d_acc, e0, e1);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(d_acc);
  return st;
}

int rdr_time_kernels(rdr_handle* h, const double* x, double* y, const double* r, double* z, int reps, double* ms,
                     void* stream) {
  if (!h || !x || !y || !r || !z || !ms || reps < 1) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timed = [&](auto launch, double* out) -> int {
    CK(launch());  // warm-up
    CK(cudaEventRecord(e0, s));
    for (int k = 0; k < reps; ++k) CK(launch());
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float t = 0;
    CK(cudaEventElapsedTime(&t, e0, e1));
    *out = (double)t / reps;
    return RDR_OK;
  };
  int st = timed([&] { return launch_apply(h->op, x, y, nullptr, nullptr, s); }, &ms[0]);
  if (!st) st = timed([&] { return launch_precond_part(0, h->pc, r, z, nullptr, nullptr, s); }, &ms[1]);
  if (!st) st = timed([&] { return launch_precond_part(1, h->pc, r, z, nullptr, nullptr, s); }, &ms[2]);
  if (!st && h->fused) {  // the PCG-mode apply the solve runs: direction update + A p + stopping test
    std::memset(h->h_sc, 0, sizeof(PcgScalars));
    h->h_sc->rtol = 0.0;
    h->h_sc->maxit = 1 << 30;  // the stopping test never fires (x != 0: ||z_0|| > 0)
    CK(cudaMemcpyAsync(h->d_sc, h->h_sc, sizeof(PcgScalars), cudaMemcpyHostToDevice, s));
    st = timed([&] { return launch_pcg_fused_apply(h->op, h->d_sc, x, h->d_p, h->d_p2, y, s); }, &ms[3]);
  } else if (!st) {
    ms[3] = 0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return st;
}

int rdr_measure_fp64_peak(double* tflops, void* stream) {
  if (!tflops) return RDR_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* d;
  CK(cudaMalloc((void**)&d, sizeof(double)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int n = 1 << 15, threads = 512;
  CK(launch_dmma_peak(d, n, sms, threads, s));  // warm-up
  CK(cudaEventRecord(e0, s));
  CK(launch_dmma_peak(d, n, sms, threads, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *tflops = 512.0 * 4.0 * n * (double)sms * (threads / 32) / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return RDR_OK;
}

void rdr_destroy(rdr_handle* h) {
  if (h) {
    cudaDeviceSynchronize();
    delete h;
  }
}

const char* rdr_strerror(int code) {
  switch (code) {
    case RDR_OK: return "ok";
    case RDR_EINVAL: return "invalid argument";
    case RDR_EMESH: return "invalid mesh (degenerate cell, non-manifold face or mask on an interior face)";
    case RDR_ENOTSPD: return "patch matrix not SPD";
    case RDR_ENOMEM: return "out of memory";
    case RDR_ECUDA: return "CUDA error";
    case RDR_ENOCONV: return "PCG did not converge within maxit";
    default: return "unknown error";
  }
}

int rdr_reference_matrices(int space, int p, double* out, int32_t* n_loc, int32_t* n_mat) {
  if (!n_loc || !n_mat) return RDR_EINVAL;
  if (space != RDR_HGRAD && space != RDR_HCURL && space != RDR_HDIV) return RDR_EINVAL;
  if (p < 1 || (space == RDR_HGRAD && p > 12) || (space != RDR_HGRAD && p > 10)) return RDR_EINVAL;
  try {
    const RefElement& el = reference_element(space, p);
    *n_loc = el.n;
    *n_mat = el.n_mat;
    if (out) std::memcpy(out, el.R.data(), sizeof(double) * el.R.size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rdr_reference_matrices: %s\n", e.what());
    return RDR_EINVAL;
  }
  return RDR_OK;
}

int rdr_reference_factors(int space, int p, double* out, int32_t* n_loc, int32_t* nf, int32_t* nfm) {
  if (!n_loc || !nf || !nfm) return RDR_EINVAL;
  if (space != RDR_HGRAD && space != RDR_HCURL && space != RDR_HDIV) return RDR_EINVAL;
  if (p < 1 || (space == RDR_HGRAD && p > 12) || (space != RDR_HGRAD && p > 10)) return RDR_EINVAL;
  try {
    const RefElement& el = reference_element(space, p);
    *n_loc = el.n;
    *nf = el.nf;
    *nfm = el.nfm;
    if (out && el.nf) std::memcpy(out, el.F.data(), sizeof(double) * el.F.size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rdr_reference_factors: %s\n", e.what());
    return RDR_EINVAL;
  }
  return RDR_OK;
}

int rdr_spd_inverse(double* a, int32_t n) {
  if (!a || n < 1) return RDR_EINVAL;
  std::vector<double> work;
  return spd_inverse(a, n, work) ? RDR_OK : RDR_ENOTSPD;
}

int rdr_bubble_eigenvalues(int kind, int l, int p, double* out, int32_t* n) {
  if (!n || kind < 0 || kind > 2 || l < 1 || l > 3 || p < 1 || p > 12 || (kind == 1 && l < 2) || (kind == 2 && l != 3))
    return RDR_EINVAL;
  try {
    std::vector<double> v = bubble_eigenvalues(kind, l, p);
    *n = (int32_t)v.size();
    if (out) std::memcpy(out, v.data(), sizeof(double) * v.size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rdr_bubble_eigenvalues: %s\n", e.what());
    return RDR_EINVAL;
  }
  return RDR_OK;
}

}  // extern "C"
