// Host-side setup of the Riesz-map operator and preconditioner (SURVEY §8(a)
// S0/S1 and the patch factorisation of P:2284-2288).
#pragma once
#include <cstdint>
#include <vector>

#include "refelem.hpp"

namespace rdr {

struct Mesh {
  int64_t nv = 0, nt = 0, ne = 0, nf = 0;
  std::vector<double> x;             // [nv][3]
  std::vector<int32_t> cells;        // [nt][4], sorted vertex ids (R-A3)
  std::vector<int32_t> cell_edges;   // [nt][6] local edge order (01,02,03,12,13,23)
  std::vector<int32_t> cell_faces;   // [nt][4] local face order (012,013,023,123)
  std::vector<int32_t> edges;        // [ne][2] lexicographic (R-A9)
  std::vector<int32_t> faces;        // [nf][3] lexicographic
  std::vector<uint8_t> dir_v, dir_e, dir_f;  // Dirichlet closure (R-A11)
};

// Returns 0 or an rdr error code (RDR_EMESH).
int build_mesh(const double* x, int64_t nv, const int32_t* tets, int64_t nt, const uint8_t* mask, Mesh& m);

struct Numbering {
  int space = 0, p = 0;
  int64_t per[4] = {0, 0, 0, 0};
  int64_t off[4] = {0, 0, 0, 0};
  int64_t n_total = 0;
  std::vector<int32_t> dofmap;       // [nt][n_loc] global ids
  std::vector<uint8_t> constrained;  // [n_total]
};

void build_numbering(const Mesh& m, const RefElement& el, Numbering& num);

// Entity form of the dof map used by the operator apply (kernels.cu): per cell
// the first global dof of each of its 15 local entities (4 vertices, 6 edges,
// 4 faces, the cell; -1 if constrained or without dofs), per cell the bits of
// the entities it owns (the lowest-index cell containing a free entity), and
// per local dof (entity << 9) | position inside the entity's block.
struct EntityMap {
  std::vector<int32_t> ebase;  // [nt][16]
  std::vector<uint16_t> own;   // [nt]
  std::vector<uint16_t> lut;   // [n_loc]
};
// Returns 0, or -1 if the dof map does not have the entity form.
int build_entity_map(const Mesh& m, const Numbering& num, const RefElement& el, EntityMap& em);

// Per-cell coefficients c_{e,s} (7 for H(grad), 12 for H(curl)), see setup.cpp.
void cell_coefficients(const Mesh& m, int space, const double* alpha, const double* beta, std::vector<double>& c);

struct Patches {
  // patches sorted by decreasing size; indices are global ids in `space_of_idx`
  // (0 = the problem's own numbering, 1 = the CG_p potential numbering)
  std::vector<int32_t> n;            // [np] patch dimension
  std::vector<int64_t> idx_off;      // [np+1] offsets into idx
  std::vector<int32_t> idx;          // patch dof ids (padded to a multiple of 32 with -1)
  std::vector<int64_t> tile_off;     // [np+1] offsets (in doubles) into the packed inverse store
  std::vector<uint8_t> kind;         // [np] 0 = direct dofs, 1 = potential (through G)
  int64_t total_doubles = 0;
  int32_t max_n = 0;
  double alg_bytes = 0;              // 8 sum n(n+1)/2
};

// Stored layout of one patch inverse A_m^{-1} (n x n, symmetric): the lower
// triangle in 32-row block rows I = 0..nb-1 (rows = min(32, n - 32 I)); block
// row I holds I full-width tiles J < I, in one of two layouts: kTileGroups
// (i,k) at ((k>>2)*rows + i)*4 + (k&3) -- 32-byte groups of 4 columns, one per
// row, for coalesced direct loads with lane = row (patch_ldg_kernel) -- or
// kTileSwizzled (i,k) at i*32 + 2*((k>>1) ^ (i&7)) + (k&1) -- 16-byte chunks
// XOR-swizzled by row, so that lane-per-row 16-byte and lane-per-column
// 8-byte reads of the tile in shared memory are both bank-conflict free
// (patch_stream_kernel)
// followed by the diagonal tile packed by columns ((i,k), k <= i, at
// k*rows - k(k-1)/2 + (i-k)). Exactly n(n+1)/2 doubles, padded to 16.
inline int64_t patch_block_row_start(int n, int I) {
  (void)n;
  return 512LL * I * I + 16LL * I;  // sum_{I'<I} (1024 I' + 528), all earlier rows are full
}
inline int64_t patch_tile_offset(int n, int I, int J) {
  const int rows = (n - 32 * I) < 32 ? (n - 32 * I) : 32;
  return patch_block_row_start(n, I) + (int64_t)J * 32 * rows;
}
inline int64_t patch_stored_doubles(int n) {
  const int64_t exact = (int64_t)n * (n + 1) / 2;
  return (exact + 15) / 16 * 16;
}

// Builds the patch index sets (R-A13; unsplit: the interiors of the star's
// cells too, Eq. 5.2 / 5.10), assembles and inverts each patch
// matrix (R-A15), and hands the packed tiles to `sink(first_patch, last_patch,
// host_tiles)` in chunks so that the full inverse store never lives on the host.
// Returns 0 or RDR_ENOTSPD.
struct PatchSink {
  virtual int reserve(int64_t total_doubles) = 0;
  virtual int put(int64_t tile_begin, const double* tiles, int64_t count) = 0;
  virtual ~PatchSink() {}
};
enum PatchLayout { kTileGroups = 0, kTileSwizzled = 1 };
// Assembly lists of the device setup (patch_setup.hpp DevPatchSetup): patch k
// has cell records [rec_ptr[k], rec_ptr[k+1]), record r is cell rec_cell[r]
// with entries ent[rec_off[r] .. rec_off[r+1]) = (local dof << 16) | position.
struct PatchAssembly {
  std::vector<int64_t> rec_ptr, rec_off;
  std::vector<int32_t> rec_cell;
  std::vector<uint32_t> ent;
};
// dev == nullptr: assemble, invert and pack on the host and hand the tiles to
// `sink`; otherwise only reserve the store and fill *dev for patch_setup.cu.
int build_patches(const Mesh& m, const Numbering& num, const RefElement& el, const std::vector<double>& coef,
                  const Numbering* cg_num, const RefElement* cg_el, const std::vector<double>* cg_coef,
                  Patches& P, PatchSink& sink, PatchLayout layout, bool unsplit = false,
                  PatchAssembly* dev = nullptr);

// Packs the symmetric n x n matrix W2 (row-major) into the patch tile layout.
void pack_patch_tiles(const double* W2, int n, double* out, PatchLayout layout);

// Whitney coarse space of the hybrid Schwarz preconditioner:
// the free vertex dofs (H(grad)) / Whitney edge dofs (H(curl)), Lemma 4.1
// P:906-989, and the stored inverse of A restricted to them, packed as one
// patch (layout kTileGroups). With `dense`, only A restricted to them (nc x nc
// row-major) is returned there, for the device inverse. Returns 0 or RDR_ENOTSPD.
int build_coarse(const Mesh& m, const Numbering& num, const RefElement& el, const std::vector<double>& coef,
                 std::vector<int32_t>& cidx, std::vector<double>& tiles, std::vector<double>* dense = nullptr);

// Interior point-Jacobi (R-A17): 1/A_ll for the cell-interior dofs [off[3], n_total).
void interior_inverse_diagonal(const Mesh& m, const Numbering& num, const RefElement& el,
                               const std::vector<double>& coef, std::vector<double>& dinv);

// Discrete gradient rows for the H(curl) potential space (R-A12), CSR over the
// CG_p dofs: g_c = sum_k G[k][c] r_k.
struct Gradient {
  std::vector<int64_t> ptr;   // [n_cg + 1]
  std::vector<int32_t> col;   // Ned1 dof ids
  std::vector<double> val;    // +-1
};
void build_gradient(const Mesh& m, const Numbering& ned, const Numbering& cg, Gradient& G);

}  // namespace rdr
