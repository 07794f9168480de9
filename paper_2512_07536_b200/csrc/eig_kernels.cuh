// GPU symmetric eigendecomposition for the API's sym_eig (eig_kernels.cu).
#pragma once

namespace tpb {

// a: n x n row-major (symmetrized internally); values ascending; vectors
// row-major with column k the eigenvector of values[k].
void sym_eig_device(int n, const double* a, double* values, double* vectors);

}  // namespace tpb
