// Reference element of the paper's basis, built on the host in x87 extended
// precision (long double) and rounded to FP64 once (DESIGN.md R-A24).
#pragma once
#include <array>
#include <string>
#include <vector>

namespace rdr {

struct LocalDof {
  int dim;    // 0 vertex, 1 edge, 2 face, 3 cell
  int ent;    // local entity index on T-hat (R-A8 order)
  int j;      // index inside the entity's family
  int type;   // 0 = type-I / vertex / H(grad) bubble, 1 = type-II, 2 = Whitney
};

struct RefElement {
  int space = 0;                 // 0 H(grad), 1 H(curl)
  int p = 0;
  int n = 0;                     // local dofs
  int n_mat = 0;                 // 7 or 12
  std::vector<LocalDof> dofs;    // R-A8 order
  std::vector<double> R;         // [n_mat][n][n] symmetric reference matrices (FP64)
  std::vector<double> lam_cell;  // interior type-I eigenvalues
  // H(curl) only: the reference matrices factored through L2-orthonormal bases of P_p (values)
  // and P_{p-1} (curls): M^{ab} = F_a^M F_b^M^T, K^{ab} = F_a^K F_b^K^T with F_a^M = P_a L_p,
  // F_a^K = Rc_a L_{p-1} (P_a, Rc_a: component a of the basis functions / their curls in the
  // barycentric monomials; L_q L_q^T the monomial Gram matrix). F = [n][nf], columns
  // [F_0^M | F_1^M | F_2^M | F_0^K | F_1^K | F_2^K], nfm = 3 dim P_p (0: not factored).
  // H(div): [F_0^M | F_1^M | F_2^M | F^D], the div-div matrix K = F^D F^D^T (one component).
  int nf = 0, nfm = 0;
  std::vector<double> F;
};

// Cached per (space, p). Throws std::runtime_error on internal failure.
const RefElement& reference_element(int space, int p);

// Bubble eigenvalues on the canonical l-simplex; kind 0 = CG_p, 1 = Ned1_p.
std::vector<double> bubble_eigenvalues(int kind, int l, int p);

}  // namespace rdr
