/* rdr.h — C ABI of the B200 Riesz-map PCG library (arXiv 2506.17406 hot path).
 *
 * Problem (Eq. 2.9): find u in X^k_{p,D} with
 *     a^k(u, v) = (u, beta v) + (d^k u, alpha d^k v) = F(v)  for all v,
 * k = 0 (H(grad), CG_p), k = 1 (H(curl), first-kind Nedelec Ned1_p,
 * P:288-299 Eq. 2.4) or k = 2 (H(div), Raviart-Thomas RT_p),
 * piecewise-constant alpha > 0, beta >= 0 per cell, on an
 * affine tetrahedral mesh, in the paper's basis (dofs = moments against
 * doubly-orthogonal bubble eigenbases, Eq. 3.8-3.10, §3.4.1-3.4.3
 * P:725-858; basis = Ciarlet dual).
 *
 * Vectors: full length n_total in the canonical global numbering of DESIGN.md
 * R-A9 (dimension-major: vertices by id, edges sorted lexicographically,
 * faces sorted, cells in input order; inside an entity R-A8). Constrained
 * (Dirichlet) entries of inputs are ignored (read as 0);
 * constrained entries of outputs are written as 0.
 *
 * Ownership: the library copies everything it needs during rdr_setup and
 * retains no caller pointer. The handle owns all device buffers; rdr_destroy
 * frees them (safe on NULL). A handle must not be used from two host threads
 * at once.
 *
 * Streams: all device work is enqueued on the stream argument (a cudaStream_t
 * passed as void*, NULL = legacy default stream). rdr_apply and rdr_precond
 * never synchronize. rdr_setup and rdr_solve synchronize the stream.
 *
 * Errors: every function returns an rdr status and never aborts. On error the
 * outputs are unspecified, except that rdr_solve returning RDR_ENOCONV still
 * writes x and sets *iters = maxit.
 */
#ifndef RDR_H
#define RDR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rdr_handle rdr_handle;

/* Spaces: H(grad) CG_p (1 <= p <= 12), H(curl) Ned1_p (1 <= p <= 10) and
 * H(div) RT_p (1 <= p <= 10, Eq. 3.17-3.18, Piola
 * pullback of 2-forms, edge-star patches PAFW1(X2_Gamma) + J(X2_I), Eq. 5.16
 * P:2156-2164; unsplit: PAFW1(X2)). */
enum { RDR_HGRAD = 0, RDR_HCURL = 1, RDR_HDIV = 2 };

/* Space decomposition of the preconditioner (both one-level additive, unit
 * weights, exact local solvers; DESIGN.md R-A13..A15):
 *   RDR_SPLIT   (default, the hot path) interface star patches + point-Jacobi
 *               on the interiors: PAFW0(X0_Gamma)+J(X0_I) (Eq. 5.4)
 *               for H(grad), PH(X0_Gamma, X1I_Gamma)+J(X1_I) (Eq. 5.12,
 *               P:1956-1970) for H(curl), PAFW1(X2_Gamma)+J(X2_I) (Eq. 5.16,
 *               edge stars) for H(div);
 *   RDR_UNSPLIT the baselines the split is measured against (NEXT-3): star
 *               patches that contain the cell interiors and no Jacobi,
 *               PAFW0(X0) (Eq. 5.2), PH(X0, X1I) (Eq. 5.10,
 *               P:1899-1905) and PAFW1(X2) -- 3439 vs 1423 dofs per vertex
 *               star at p = 10. */
enum { RDR_SPLIT = 0, RDR_UNSPLIT = 1 };

/* Composition of the preconditioner:
 *   RDR_ADDITIVE (default, the hot path) one-level additive J(X_I) + patches;
 *   RDR_HYBRID   the paper's symmetric multiplicative hybrid Schwarz (P:2399-2455,
 *                NEXT-1): sweep X_I (Jacobi), X_Gamma (additive patches),
 *                W^k (exact solve on the Whitney space: vertex dofs for H(grad),
 *                Whitney edge dofs for H(curl), Whitney face dofs for H(div),
 *                Lemma 4.1; its inverse is formed on the device), X_Gamma, X_I, each
 *                damped by rho_m = (lambda_min + 3 lambda_max)/4 from 10 CG-Lanczos
 *                steps. Split decomposition only; costs 4 extra
 *                operator applies per preconditioner application. */
enum { RDR_ADDITIVE = 0, RDR_HYBRID = 1 };

/* Where the star-patch matrices are assembled and inverted at setup (SURVEY
 * NEXT-4; the patch factorisation of P:2284-2288):
 *   RDR_SETUP_DEVICE (default) -- on the GPU (patch_setup.cu): per-CTA block
 *                Gauss-Jordan sweep of each patch matrix in device scratch,
 *                written straight into the stored tile layout;
 *   RDR_SETUP_HOST -- on the host cores (blocked Cholesky-based inverse,
 *                dense.cpp), then uploaded. Both give A_m^-1 to rounding. */
enum { RDR_SETUP_DEVICE = 0, RDR_SETUP_HOST = 1 };

/* How rdr_solve drives the PCG iteration (R-A16); all of them run the same
 * arithmetic and give the same iterates (to rounding):
 *   RDR_LOOP_DEVICE (default) -- the loop runs on the device with one host
 *                synchronisation per solve: small problems (additive
 *                preconditioner, star patches <= 256 dofs, n_loc <= 128) as one
 *                persistent cooperative kernel when a 40-iteration solve timed
 *                at setup is faster that way (rdr_info.persistent_loop), else as
 *                RDR_LOOP_GRAPH;
 *   RDR_LOOP_HOST -- graphs of 8 iterations relaunched by the host until done;
 *   RDR_LOOP_EAGER -- every kernel launched on the stream, the host testing the
 *                stop flag after each iteration (no graphs: profilers see every
 *                kernel of the iteration);
 *   RDR_LOOP_GRAPH -- one CUDA graph whose conditional WHILE node repeats a body
 *                of 8 iterations (3 kernels each: fused apply with the stopping
 *                test, update + Jacobi, patches) until the test fires (the
 *                hybrid preconditioner: a body of one unfused iteration, its
 *                sweep included, so nothing runs past convergence);
 *   RDR_LOOP_PERSISTENT -- the whole solve in one persistent cooperative kernel
 *                (grid barriers between the phases of each iteration; CUDA-core
 *                apply with the reference matrices in shared memory, one warp
 *                per patch); RDR_EINVAL at setup if the problem is not eligible. */
enum { RDR_LOOP_DEVICE = 0, RDR_LOOP_HOST = 1, RDR_LOOP_EAGER = 2, RDR_LOOP_GRAPH = 3, RDR_LOOP_PERSISTENT = 4 };

struct rdr_options {
  int decomposition;  /* RDR_SPLIT or RDR_UNSPLIT */
  int preconditioner; /* RDR_ADDITIVE or RDR_HYBRID */
  int setup;          /* RDR_SETUP_DEVICE or RDR_SETUP_HOST */
  int loop;           /* RDR_LOOP_DEVICE, _HOST, _EAGER, _GRAPH or _PERSISTENT */
};

enum {
  RDR_OK = 0,
  RDR_EINVAL = -1,   /* bad p / space / sizes / options / NULL pointer; alpha <= 0, beta < 0, or
                        beta = 0 with H(curl) or H(div) (gradients resp. div-free fields
                        would be in the kernel of A and of the star-patch matrices) */
  RDR_EMESH = -2,    /* |det J| <= 1e-12 h^3, non-manifold face, mask bit on an interior face */
  RDR_ENOTSPD = -3,  /* a non-positive pivot while inverting a patch (or the hybrid coarse) matrix */
  RDR_ENOMEM = -4,   /* device or host allocation failed */
  RDR_ECUDA = -5,    /* any other CUDA runtime error */
  RDR_ENOCONV = -6   /* PCG reached maxit */
};

struct rdr_info {
  int64_t n_total;       /* vector length (all dofs, constrained included) */
  int64_t n_free;        /* unconstrained dofs */
  int64_t n_interior;    /* cell-interior dofs (point-Jacobi block, Thm 5.1) */
  int64_t n_cells;
  int32_t n_loc;         /* local dofs per cell */
  int32_t n_mat;         /* reference matrices: 7 (H(grad), H(div)) or 12 (H(curl)) */
  int64_t n_patches;     /* star patches (Eq. 5.4 P:1763-1774 / Eq. 5.12) */
  int32_t max_patch;     /* largest patch dimension */
  int64_t patch_bytes;   /* device bytes of the stored patch inverses (with tile padding) */
  double flops_apply;    /* algorithmic flops of one rdr_apply: 2 n_loc^2 n_mat n_cells */
  double bytes_apply;    /* algorithmic HBM bytes of one rdr_apply */
  double bytes_precond;  /* algorithmic HBM bytes of one rdr_precond: 8 sum n_m(n_m+1)/2 + 24 N_int */
  double setup_seconds;  /* wall time of rdr_setup */
  double refelem_seconds;      /* of which: reference element construction (cached per process) */
  double patch_setup_seconds;  /* of which: patch index sets, assembly, inversion and packing */
  double patch_kernel_seconds; /* of which: the device assembly + inversion kernel (RDR_SETUP_DEVICE), else 0 */
  double patch_setup_flops;    /* algorithmic flops of the device block sweep: per patch, with
                                  nb = ceil(n/64), sum over pivot blocks of 2*64^3 per updated
                                  lower tile and panel product = 2*64^3 nb (nb-1)(nb+2)/2 */
  int32_t apply_variant;       /* warp layout of the operator apply chosen by setup-time autotuning */
  int32_t apply_grid;          /* its persistent grid (CTAs) */
  int32_t persistent_loop;     /* 1: solves run as the persistent cooperative kernel (RDR_LOOP_DEVICE
                                  chose it, or RDR_LOOP_PERSISTENT) */
  int32_t apply_slots;         /* its TMA ring depth (reference-stack chunks of n_mat KB) */
  int32_t small_patch_grid;    /* > 0: all patches <= 128 dofs and setup's timing chose resident warps
                                  walking them (this many CTAs); 0: one warp per patch or CTA per patch */
  int32_t apply_factored;      /* 1 / 2 / 3: the apply runs factored through orthonormal P_p / P_{p-1} bases
                                  with (16, 16) / (32, 32) / (32, 24) cells per tile of its two stages
                                  (two-stage kernels, H(curl) and H(div)), chosen by setup-time
                                  timing against the DMMA apply with the reference matrices */
  int32_t apply_fact_split_a;  /* factored apply: CTAs per cell tile in stage A (each a share of the 32-column */
  int32_t apply_fact_split_b;  /* blocks of U) and in stage B (of Y), chosen by the same timing; 0 if not factored */
};

/* Build the operator and the preconditioner (host setup once, then upload).
 *   vertices [nv][3] float64 row-major; tets [nt][4] int32 (any vertex order);
 *   alpha, beta [nt] float64; dirichlet_mask [nt][4] uint8: bit (t,i) = 1 iff
 *   the face opposite INPUT vertex i of tet t lies on Gamma_D.
 *   Each of these five pointers may be host or device memory (detected).
 *   1 <= p <= 12 for H(grad), 1 <= p <= 10 for H(curl) and H(div).
 *   Reference element: DESIGN.md readings R-A1..A8, R-A24 (extended precision,
 *   P:595-619). Patches: R-A13. Inverses stored per patch (R-A15). */
int rdr_setup(rdr_handle** h, const double* vertices, int64_t nv, const int32_t* tets, int64_t nt,
              int p, int space, const double* alpha, const double* beta,
              const uint8_t* dirichlet_mask, void* stream);

/* rdr_setup with options (NULL = defaults: RDR_SPLIT, RDR_ADDITIVE,
 * RDR_SETUP_DEVICE, RDR_LOOP_DEVICE). RDR_EINVAL for an unknown decomposition,
 * preconditioner, setup or loop, or RDR_HYBRID with RDR_UNSPLIT. */
int rdr_setup_ex(rdr_handle** h, const double* vertices, int64_t nv, const int32_t* tets, int64_t nt,
                 int p, int space, const double* alpha, const double* beta,
                 const uint8_t* dirichlet_mask, const struct rdr_options* opt, void* stream);

int rdr_ndofs(const rdr_handle* h, int64_t* n_total);
/* rho[3]: the hybrid Schwarz weights rho_1 (interior Jacobi), rho_2 (patches), rho_3 = 1 (coarse). */
int rdr_get_weights(const rdr_handle* h, double* rho);
int rdr_get_info(const rdr_handle* h, struct rdr_info* out);

/* y = A x (device pointers, length n_total): gather, per-cell contraction
 * y_e = sum_s c_{e,s} R_s x_e with the shared reference matrices, scatter-add
 * (north_star; matrix-free action P:2267-2275). */
int rdr_apply(rdr_handle* h, const double* x, double* y, void* stream);

/* z = P^-1 r (device pointers): interior point-Jacobi + additive star patches
 * (DESIGN.md R-A13..A17). */
int rdr_precond(rdr_handle* h, const double* r, double* z, void* stream);

/* PCG (DESIGN.md R-A16) from x0 = 0 on device vectors b -> x.
 * *iters (host) receives the iteration count; synchronizes `stream`. */
int rdr_solve(rdr_handle* h, const double* b, double* x, double rtol, int maxit, int* iters, void* stream);

/* Same as rdr_solve with HOST b and x (pinned or pageable): H2D copy of b,
 * PCG, D2H copy of x, all on `stream` (the end-to-end path). */
int rdr_solve_host(rdr_handle* h, const double* b_host, double* x_host, double rtol, int maxit,
                   int* iters, void* stream);

/* Per-kernel launch accounting of the last rdr_solve: number of library kernel
 * launches (graph nodes included). */
int rdr_last_launches(const rdr_handle* h, int64_t* launches);

/* Outcome of the last rdr_solve / rdr_solve_host / rdr_profile_solve:
 * iterations, whether the stopping test ||z_k|| <= rtol ||z_0|| (R-A16) fired,
 * ||z_0|| and ||z_k|| at the last test, and the kernel launches. */
struct rdr_solve_stats {
  int32_t iters;
  int32_t converged;
  double z0;
  double z_last;
  int64_t launches;
};
int rdr_last_solve(const rdr_handle* h, struct rdr_solve_stats* out);

/* Measurement helper: one PCG solve (as rdr_solve, x left in the handle)
 * with every kernel launched eagerly and CUDA events between the kernel groups
 * of each iteration; ms[4] receives the average device ms per iteration of
 * ms[0] the fused operator apply (direction update + A p + stopping test),
 * ms[1] the x/r update + interior Jacobi, ms[2] the star-patch solves
 * (H(curl): the discrete gradient of the potential patches included),
 * ms[3] = 0 -- the in-solve counterparts of rdr_time_kernels ms[0..2]. Additive preconditioner only
 * (RDR_EINVAL otherwise). Synchronizes `stream`. */
int rdr_profile_solve(rdr_handle* h, const double* b, double rtol, int maxit, int* iters, double* ms,
                      void* stream);

/* Measurement helper: the SM clock the fused apply runs at, inside the PCG
 * iteration and alone. A PCG on b (device, n_total) is run for `iters` timed
 * iterations with rtol 0 (stream launches, no host synchronisation in
 * between), with a one-thread probe kernel behind each fused apply that spins
 * 10 us of %globaltimer and reads clock64; then the fused apply is launched
 * `iters` times back to back with the same probe. out[4] (host): out[0] mean
 * SM MHz behind the apply in the iteration, out[1] the same for the apply
 * alone, out[2] ms per iteration (probe time subtracted), out[3] ms per apply
 * alone. Additive preconditioner only (RDR_EINVAL otherwise). Synchronizes
 * `stream`; the handle's solve vectors are overwritten. */
int rdr_debug_profile_clocks(rdr_handle* h, const double* b, int iters, double* out, void* stream);

/* Measurement helper (bench.py roofline): launch each hot-path kernel `reps`
 * times back to back on `stream` between CUDA events and return the average
 * device time per launch in ms: ms[0] operator apply (gather-contract-scatter),
 * ms[1] interior Jacobi + zeroing, ms[2] patch solves (H(curl): with the
 * discrete gradient of the potential patches), ms[3] the fused PCG-mode apply
 * the solve runs (direction update + A p + stopping test; 0 with the hybrid
 * preconditioner, whose PCG uses the plain apply). x must be nonzero on free dofs. x, r: device input vectors, y, z: outputs
 * (contents overwritten). Synchronizes `stream`. */
int rdr_time_kernels(rdr_handle* h, const double* x, double* y, const double* r, double* z, int reps, double* ms,
                     void* stream);

/* Measurement helper (bench.py roofline denominator of the apply): FP64
 * tensor-core (DMMA.8x8x4) throughput of an issue-bound loop over all SMs, in
 * TFLOP/s, timed with CUDA events on `stream` (synchronizes it). */
int rdr_measure_fp64_peak(double* tflops, void* stream);

void rdr_destroy(rdr_handle* h);
const char* rdr_strerror(int code);

/* Debugging entry point: run the operator apply (and the solves) with warp
 * layout `variant` (0 <= variant < 18; kernels.cu apply_variants) instead of the
 * one setup's autotuning chose; RDR_EINVAL if it does not fit this operator.
 * The GPU tests use it to check every layout against the oracle. */
int rdr_debug_set_apply_variant(rdr_handle* h, int variant);

/* Debugging entry point: the apply's warp layout `variant` with a ring of
 * `slots` reference-stack chunks and a grid of `grid` CTAs (0: the persistent
 * grid of resident CTAs) -- the three values rdr_info reports as apply_variant,
 * apply_slots and apply_grid -- so that a profiler run can reproduce the
 * configuration another setup's timing chose (scripts/prof_kernels.py --apply);
 * variant = -1 / -2 / -3 selects the factored two-stage apply with (16, 16) / (32, 32) / (32, 24)
 * cells per tile of its two stages (H(curl), H(div); rdr_info.apply_factored = 1 / 2 / 3), with
 * `slots` / `grid` (0..8, 0 = 1) CTAs per cell tile in stage A / stage B (rdr_info.apply_fact_split_a / _b).
 * RDR_EINVAL if it does not fit this operator. */
int rdr_debug_set_apply_config(rdr_handle* h, int variant, int slots, int grid);

/* Debugging entry point: run the small star patches (configurations whose
 * patches all have <= 128 dofs, e.g. the H(div) edge stars) with one warp per
 * patch (persistent = 0) or with resident warps that walk the patches and load
 * the next one's tiles while scattering the current one (persistent = 1)
 * instead of the one setup's timing chose; RDR_EINVAL if the configuration
 * has no small-patch launch. */
int rdr_debug_set_small_patch_kernel(rdr_handle* h, int persistent);

/* Debugging entry point: one fused PCG operator apply at iteration 0 (q = A z
 * through the PCG variant of the apply kernel, which also writes the search
 * direction); compared against rdr_apply by the GPU tests. Synchronizes. */
int rdr_debug_fused_apply(rdr_handle* h, const double* z, double* q, void* stream);

/* Host-only debug entry points (no device needed).
 * rdr_reference_matrices: the n_mat reference matrices of (space, p) in
 * float64, layout [n_mat][n_loc][n_loc]; pass out = NULL to query *n_loc and
 * *n_mat. Order: H(grad) M, Kxx, Kyy, Kzz, Kxy+Kyx, Kxz+Kzx, Kyz+Kzy;
 * H(curl) Mxx, Myy, Mzz, Mxy+Myx, Mxz+Mzx, Myz+Mzy, then the same for K (curl);
 * H(div) Mxx, Myy, Mzz, Mxy+Myx, Mxz+Mzx, Myz+Mzy (2-form proxies), then K (div-div).
 * Local dof order: DESIGN.md R-A8. */
int rdr_reference_matrices(int space, int p, double* out, int32_t* n_loc, int32_t* n_mat);
/* rdr_reference_factors (H(curl), H(div)): the factors of the reference matrices
 * through L2-orthonormal bases of P_p (values) and P_{p-1} (curls / divergences)
 * that the factored apply uses, layout [n_loc][nf]. H(curl): columns
 * [F0M | F1M | F2M | F0K | F1K | F2K] with nfm = 3 dim P_p, M^{ab} = FaM FbM^T,
 * K^{ab} = FaK FbK^T; H(div): [F0M | F1M | F2M | FD], K = FD FD^T (DESIGN.md
 * section 10e). Pass out = NULL to query *n_loc, *nf and *nfm; *nf = 0 for H(grad). */
int rdr_reference_factors(int space, int p, double* out, int32_t* n_loc, int32_t* nf, int32_t* nfm);
/* In-place inverse of an n x n SPD row-major matrix with the host routine the
 * setup uses for the patch inverses (R-A15); RDR_ENOTSPD on a non-positive
 * Cholesky pivot. */
int rdr_spd_inverse(double* a, int32_t n);
/* Bubble eigenvalues lambda_j (Eq. 3.8) on the canonical l-simplex: kind 0 = CG, 1 = Ned1,
 * 2 = RT (l = 3 only, Eq. 3.17). */
int rdr_bubble_eigenvalues(int kind, int l, int p, double* out, int32_t* n);

#ifdef __cplusplus
}
#endif
#endif
