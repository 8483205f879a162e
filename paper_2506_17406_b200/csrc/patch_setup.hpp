// Device-side patch setup: the star-patch matrices
// A_m = sum_{T in star(m)} E_T^T A_T E_T (element matrices of Eq. 2.9 from the
// shared reference matrices, DESIGN.md R-A10) are assembled and inverted on the
// GPU and written straight into the stored tile layout of setup.hpp -- the
// patch factorisation of P:2284-2288 done once at setup, without the host
// O(sum n_m^3) loop or the upload of the inverse store.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rdr {

struct DevPatchSetup {
  int64_t np = 0;
  const int32_t* pn = nullptr;        // [np] patch dimension n_m
  const uint8_t* pkind = nullptr;     // [np] 0: own numbering, 1: CG potential numbering (H(curl) vertex stars)
  const int64_t* tile_off = nullptr;  // [np+1] offsets (doubles) into `tiles`
  double* tiles = nullptr;            // packed inverse store (setup.hpp layout `layout`)
  int layout = 0;                     // PatchLayout: 0 kTileGroups, 1 kTileSwizzled
  // assembly lists: patch k has cell records [rec_ptr[k], rec_ptr[k+1]); record
  // r is cell rec_cell[r] with entries ent[rec_off[r] .. rec_off[r+1]), each
  // (local dof << 16) | position in the patch
  const int64_t* rec_ptr = nullptr;
  const int32_t* rec_cell = nullptr;
  const int64_t* rec_off = nullptr;
  const uint32_t* ent = nullptr;
  // per numbering kind: reference matrices [nm][nl][nl] and cell coefficients [nt][nm]
  const double* R[2] = {nullptr, nullptr};
  const double* coef[2] = {nullptr, nullptr};
  int nl[2] = {0, 0}, nm[2] = {0, 0};
  double* scratch = nullptr;  // per CTA: patch_setup_scratch_doubles(ld_max)
  int64_t ld_max = 0;         // max n_m rounded up to 64
  int32_t* queue = nullptr;   // [1] patch claim counter (zeroed by the caller)
  int32_t* status = nullptr;  // [1] 0, or 1 + index of a patch with a non-positive pivot (not SPD)
};

int64_t patch_setup_scratch_doubles(int64_t ld_max);
size_t patch_setup_smem();
// persistent kernel, n_ctas CTAs each claiming patches in order (largest first)
cudaError_t launch_patch_setup(const DevPatchSetup& s, int n_ctas, cudaStream_t stream);

// One large SPD matrix (the hybrid's Whitney coarse space) by the
// same block sweep with every phase spread over the grid. A: device, ld x ld
// row-major (ld = n rounded up to 64), lower triangle of A in rows/columns < n,
// zero elsewhere; destroyed. work: 64*64 + 2*64*ld doubles. *status (device,
// zeroed by the caller) becomes 1 + pivot block of a non-positive pivot.
// tiles: patch_stored_doubles(n) doubles, receives A^-1 in the layout `layout`.
cudaError_t dense_spd_inverse_packed(double* A, int64_t ld, int n, double* work, int32_t* status, double* tiles,
                                     int layout, cudaStream_t stream);

}  // namespace rdr
