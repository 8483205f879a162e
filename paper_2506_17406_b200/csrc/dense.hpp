// Host dense kernels of the setup (dense.cpp).
#pragma once
#include <vector>

namespace rdr {

// In-place inverse of a symmetric positive definite n x n row-major matrix
// (both triangles on output). `work` is resized to n*n. Returns false when a
// Cholesky pivot is not positive (RDR_ENOTSPD).
bool spd_inverse(double* A, int n, std::vector<double>& work);

}  // namespace rdr
