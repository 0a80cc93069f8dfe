// sparse_access.hpp -- internal constructors for SparseMatrix used by the
// host layer (fast CSR ingestion in the C ABI, scaled copies downloaded from
// the device).  Not part of the public API.
#pragma once

#include <vector>

#include "folp/sparse_matrix.hpp"

namespace folp {

struct SparseMatrixAccess {
  // From a valid CSR (columns strictly increasing inside each row, no
  // zeros); the column mirror (the layout from_triplets produces) is built
  // on first use.
  static SparseMatrix build(Index m, Index n, std::vector<Index> start, std::vector<Index> cols,
                            std::vector<double> vals);
  // Same structure as k, new values (CSR and CSC order).
  static SparseMatrix with_values(const SparseMatrix& k, std::vector<double> csr,
                                  std::vector<double> csc);
};

}  // namespace folp
