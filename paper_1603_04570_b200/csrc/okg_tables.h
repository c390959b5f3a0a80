// okg_tables.h -- host-side construction of the per-class stencil rows.
//
// The reference assembles M, K and b from element matrices
// (assembly.hpp:82-138) into CSR by stably sorting triplets, so every entry is
// the sum of its element contributions in ascending cell order.  Here the
// same element formulas are evaluated on the 3^d-vertex patch of a 2^d-cell
// unit grid (h = 1), in the same cell order and the same arithmetic, and the
// row of the patch vertex with boundary class c gives the stencil of every
// vertex of that class.  Scaling by h^d (M, b) and h^(d-2) (K) is exact for
// power-of-two n, so on those grids the fine-level rows are bit-identical to
// the reference's CSR rows.
#pragma once
#include <vector>

namespace okg {

struct UnitTables {
  int dim = 0;
  int ncls = 0, noff = 0;
  std::vector<double> M, K;  // [ncls][noff], unit grid
  std::vector<double> load;  // [ncls], unit grid
};

UnitTables build_unit_tables(int dim);

// dense n x n Cholesky (dense.hpp:175-196) and inverse via solves (dense.hpp:197-226);
// returns false if not positive definite.
bool dense_spd_inverse(const std::vector<double>& A, int n, std::vector<double>& inv);

// cyclic Jacobi eigenvalues of a symmetric matrix, ascending (eig.hpp:216-261);
// returns false on non-convergence.
bool symmetric_eigenvalues(std::vector<double> A, int n, std::vector<double>& ev);

}  // namespace okg
