// Launch wrappers of the sm_100a kernels (kernels.cu). Host code never sees
// device code; every wrapper enqueues on the given stream and returns the
// cudaError_t of the launch.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace rdr {

struct PcgScalars {
  double rz;       // r.z of the current iterate
  double rz_new;   // accumulator for the next r.z
  double pq;       // accumulator for p.Aq
  double zz;       // accumulator for ||z||^2
  double z0;       // ||z_0||
  double rtol;
  double beta;
  int32_t iters;
  int32_t maxit;
  int32_t done;
  int32_t converged;
  uint32_t ticket;  // last-block counter of the reduction kernel
  int32_t k;        // fused path: iteration index of the next fused apply
  double rz_acc;    // fused path: r.z accumulated by the preconditioner
  double rz_old;    // fused path: r.z of the z used by the current direction
  double pq2[2];    // fused path: p.Ap, double-buffered by iteration parity
  double z_last;    // ||z_k|| at the last stopping test (rdr_last_solve)
  // persistent PCG kernel (small problems): r.z by iteration mod 3, ||z||^2 and p.Ap by parity
  double prz[3];
  double pzz[2];
  double ppq[2];
};

struct DevOperator {
  int n_loc, n_mat;
  int64_t n_cells, n_total;
  const int32_t* ebase;         // [n_cells][16] first global dof of each local entity, -1 if constrained
                                // (setup.hpp EntityMap)
  const uint16_t* own;          // [n_cells] bit l: this cell owns local entity l (first cell containing it)
  const uint16_t* lut;          // [n_loc] (local entity << 9) | position inside the entity's block
  const double* coef;           // [n_cells][n_mat]
  const double* R;              // [n_mat][n_loc][n_loc] reference matrices (the persistent PCG kernel)
  int kp;                       // n_loc rounded up to 4: rows per reference matrix in the K stack
  int ngroups;                  // ceil(n_loc / 32) column groups
  const double* Bsw;            // [ngroups][kp/4][n_mat][4][32]: the reference matrices stacked j-major
                                // (chunk j4 = rows 4 j4 .. 4 j4 + 3 of every R_s), columns swizzled (kernels.cu
                                // apply_tc_kernel), in the local order of lut_tc
  const uint16_t* lut_tc;       // [n_loc] lut in the DMMA apply's local order: H(curl) (H(div)) puts the ncb dofs
                                // whose curl (divergence) is not zero first
  int ncb;                      // H(curl) / H(div): the curl (div-div) matrices R_s, s >= nm0, vanish outside
                                // rows / columns [0, ncb) of that order; n_loc for H(grad)
  int nm0;                      // 6 (H(curl), H(div)) or n_mat (H(grad)): the DMMA apply variants built for it
  // launch configuration (configure_apply): warp-layout variant, cell tiles, persistent grid
  int av, ntiles, apply_grid, apply_slots;
  // factored apply (H(curl)): F [kp][nfp] (RefElement::F, zero-padded),
  // nf = its columns (nfm of them the value block), ubuf [n_cells][nfp] stage-A output;
  // fact = 1 / 2 / 3: rdr_apply and the fused PCG run the two-stage factored kernels with (stage A, stage B)
  // tiles of (16, 16) / (32, 32) / (32, 24) cells
  const double* F;
  int nf, nfm, nfp, fact;
  int fact_nsa, fact_nsb;       // column splits of a cell tile over CTAs in stage A / stage B (grid.y; 0 = 1)
  int fck;                      // components of the second factor block: 3 (curls), 1 (divergence)
  double* ubuf;
};

// Meshes below this many cells keep the reference element's own rounding of the
// operator: setup does not consider the factored apply there, nor the skipped zero
// blocks of the DMMA apply (both gain nothing on such launch-bound meshes, and with a 1e4
// coefficient contrast two roundings of the same operator can move a PCG count by 2,
// profiles/round2/experiments/fact_apply_rounding.txt, skip_rounding_small.txt).
constexpr int64_t kFactMinCells = 2048;

struct DevPrecond {
  int64_t n_total, off3;        // interior dofs are [off3, n_total)
  const double* dinv;           // [n_total - off3]
  int64_t n_patches;
  int32_t max_n;                // largest patch dimension
  const int32_t* pn;            // [np]
  const int64_t* idx_off;       // [np+1]
  const int32_t* idx;
  const int64_t* tile_off;      // [np+1]
  const double* tiles;
  const uint8_t* pkind;         // 0 own numbering, 1 CG potential
  int32_t ldg_warps;            // warps per CTA of patch_ldg_kernel: 8, or 4 when most patches are small
  int64_t n_big;                // patch_ldg_kernel: patches [0, n_big) one per CTA, the rest (n <= 128) one per warp
  int32_t small_grid;           // > 0: the small patches run as patch_warp_loop_kernel on this many resident CTAs
  int32_t npad_max;             // largest patch dimension rounded up to 32
  // H(curl) potential patches: CSR rows of G^T over the CG dofs [0, n_cg_iface) they use (R-A12)
  int64_t n_cg_iface;
  const int64_t* g_ptr;
  const int32_t* g_col;
  const double* g_val;
  double out_scale;             // patch corrections are scaled by this (1; 1/rho_2 in the hybrid sweep)
  // hybrid Schwarz: Whitney coarse space and sweep workspace
  int hybrid;                   // 0 additive (J + patches), 1 symmetric multiplicative J,P,C,P,J
  double s1, s2;                // 1/rho_1 (interior Jacobi), 1/rho_2 (interface patches)
  int64_t nc;                   // coarse dofs
  const int32_t* cidx;          // [nc] their global ids
  const double* ctiles;         // packed inverse of A restricted to W^k (patch tile layout)
  double* czc;                  // [nc] coarse correction accumulators
  double* ht;                   // [n_total] sweep residual r - A e
  double* hy;                   // [n_total] A e
};

cudaError_t launch_apply(const DevOperator& op, const double* x, double* y, double* pq_acc,
                         const PcgScalars* guard, cudaStream_t s);
cudaError_t launch_precond(const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                           const PcgScalars* guard, cudaStream_t s);
// one piece of the preconditioner: 0 interior Jacobi + zeroing of the patch
// part, 1 the patch solves (H(curl) potential patches through G inside)
cudaError_t launch_precond_part(int part, const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                                const PcgScalars* guard, cudaStream_t s);
// z = P^-1 r with the hybrid sweep J, P, C, P, J (pc.hybrid = 1); needs the operator for the residuals
cudaError_t launch_precond_hybrid(const DevOperator& op, const DevPrecond& pc, const double* r, double* z,
                                  const PcgScalars* guard, cudaStream_t s);
int count_hybrid_launches(const DevPrecond& pc);
// set the while-node condition of a device-side PCG graph: continue while !sc->done
cudaError_t launch_pcg_loop_condition(const PcgScalars* sc, cudaGraphConditionalHandle loop, cudaStream_t s);
// sc->rz_new += r.z
cudaError_t launch_pcg_rz(PcgScalars* sc, const double* r, const double* z, int64_t n, cudaStream_t s);

// PCG pieces (DESIGN.md R-A16)
cudaError_t launch_pcg_init(const double* b, const uint8_t* constrained, int64_t n, double* x, double* r,
                            double* q, cudaStream_t s);
cudaError_t launch_pcg_start(PcgScalars* sc, const double* z, double* p, int64_t n, double rtol, int maxit,
                             cudaStream_t s);
cudaError_t launch_pcg_update(PcgScalars* sc, const double* p, const double* q, double* x, double* r, int64_t n,
                              cudaStream_t s);
// r != nullptr: also r.z into sc->rz_new (the hybrid preconditioner does not accumulate it)
cudaError_t launch_pcg_finish(PcgScalars* sc, const double* z, const double* r, int64_t n, cudaStream_t s);
cudaError_t launch_pcg_direction(PcgScalars* sc, const double* z, double* p, double* q, int64_t n, cudaStream_t s);

// Fused PCG step (3 kernels per iteration for H(grad)): fused apply (direction
// update + A p + ||z||^2 + stopping test), update + interior Jacobi, patches.
bool fused_pcg_supported(const DevOperator& op);
bool fact_apply_fits(const DevOperator& op, int fact);  // the factored apply's (op.fact = 1, 2, 3) shared memory fits
// setup-time choice of op.fact, timed on whole PCG iterations (b: right-hand side, cons: constrained flags,
// x, r, z, q, p0, p1: the solve's vectors, sc_init: host scalars with rtol 0 and a huge maxit)
int tune_fact(DevOperator& op, const DevPrecond& pc, const double* b, const uint8_t* cons, double* x, double* r,
              double* z, double* q, PcgScalars* sc, const PcgScalars* sc_init, double* p0, double* p1,
              cudaStream_t s, int reps);
// the apply's warp-layout variants (kernels.cu apply_variants): configure op for
// variant k (0, or -1 if it does not fit this operator), and setup-time
// autotuning over all that fit (x, y: device scratch of length n_total)
int apply_variant_count();
int apply_configure_variant(DevOperator& op, int k);
int apply_configure_exact(DevOperator& op, int k, int slots, int grid);
int tune_apply(DevOperator& op, const double* x, double* y, PcgScalars* sc, double* p0, double* p1, cudaStream_t s,
               int reps);
// setup-time choice between the two small-patch kernels (r, z: device scratch of length n_total)
int tune_small_patches(DevPrecond& pc, const double* r, double* z, cudaStream_t s, int reps);
cudaError_t launch_pcg_fused_apply(const DevOperator& op, PcgScalars* sc, const double* z, double* p0, double* p1,
                                   double* q, cudaStream_t s);
cudaError_t launch_pcg_update_jacobi(PcgScalars* sc, const DevPrecond& pc, const double* p0, const double* p1,
                                     double* q, double* x, double* r, double* z, cudaStream_t s);

// Persistent PCG (small problems, fused additive path): the whole solve of R-A16 in one
// cooperative launch -- init, then per iteration the fused apply (CUDA cores, reference
// matrices in shared memory), update + Jacobi and the warp-per-patch solves, separated by
// grid barriers. x, r, z, p0, p1, q: the handle's vectors; sc zeroed except rtol / maxit.
struct PersistentPcg {
  int warps = 0;       // warps per CTA
  int grid = 0;        // co-resident CTAs (0: not eligible)
  int wb = 0;          // per-warp scratch doubles (x 2)
  size_t smem = 0;
};
PersistentPcg plan_persistent_pcg(const DevOperator& op, const DevPrecond& pc);
cudaError_t launch_persistent_pcg(const PersistentPcg& plan, const DevOperator& op, const DevPrecond& pc,
                                  PcgScalars* sc, const double* b, const uint8_t* cons, double* x, double* r,
                                  double* z, double* p0, double* p1, double* q, cudaStream_t s);

int count_precond_launches(const DevPrecond& pc);  // kernels per rdr_precond
size_t max_kernel_smem();                           // per-CTA dynamic shared-memory opt-in used
void configure_kernels();                            // shared-memory opt-ins (call once, outside capture)
// DMMA.8x8x4 issue-bound loop: n iterations x 4 chains x 512 flop per warp
cudaError_t launch_dmma_peak(double* out, int n, int blocks, int threads, cudaStream_t s);
cudaError_t launch_sm_clock_probe(double* acc, unsigned ns, cudaStream_t s);  // acc[0] += MHz, acc[1] += 1

}  // namespace rdr
