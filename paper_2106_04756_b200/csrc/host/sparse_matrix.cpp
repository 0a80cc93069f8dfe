// sparse_matrix.cpp -- SparseMatrix construction (host) and its numerical
// methods (B200 engine).  Semantics follow
// /root/reference/proj/src/sparse_matrix.cpp (line numbers cited per method).
#include "folp/sparse_matrix.hpp"

#include <algorithm>
#include <cmath>
#include <random>

#include "device.hpp"
#include "folp/linalg.hpp"
#include "sparse_access.hpp"

namespace folp {

// from_triplets (sparse_matrix.cpp:36-104): range/finiteness checks, sort by
// (row, col), duplicates summed in sorted order, exact zeros dropped, then the
// column-compressed mirror by a counting pass.
SparseMatrix SparseMatrix::from_triplets(Index num_rows, Index num_cols,
                                         std::span<const Triplet> triplets) {
  if (num_rows < 0 || num_cols < 0) {
    throw DimensionMismatch("sparse matrix dimensions must be nonnegative");
  }
  for (const Triplet& t : triplets) {
    if (t.row < 0 || t.row >= num_rows || t.col < 0 || t.col >= num_cols) {
      throw DimensionMismatch("triplet index out of range");
    }
    if (!std::isfinite(t.value)) throw std::invalid_argument("triplet value must be finite");
  }
  std::vector<Triplet> order(triplets.begin(), triplets.end());
  std::sort(order.begin(), order.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });

  std::vector<Index> start(static_cast<std::size_t>(num_rows) + 1, 0);
  std::vector<Index> cols;
  std::vector<double> vals;
  cols.reserve(order.size());
  vals.reserve(order.size());
  for (std::size_t k = 0; k < order.size();) {
    const Index r = order[k].row, c = order[k].col;
    double sum = 0.0;
    for (; k < order.size() && order[k].row == r && order[k].col == c; ++k) sum += order[k].value;
    if (sum == 0.0) continue;
    cols.push_back(c);
    vals.push_back(sum);
    ++start[static_cast<std::size_t>(r) + 1];
  }
  for (Index r = 0; r < num_rows; ++r) start[r + 1] += start[r];
  return SparseMatrixAccess::build(num_rows, num_cols, std::move(start), std::move(cols),
                                   std::move(vals));
}

void SparseMatrix::multiply(std::span<const double> x, std::span<double> out) const {
  if (static_cast<Index>(x.size()) != num_cols_ || static_cast<Index>(out.size()) != num_rows_) {
    throw DimensionMismatch("multiply: size mismatch");
  }
  if (num_rows_ == 0) return;
  device::Context ctx(*this);
  device::check(folp_gpu_multiply(ctx.get(), 0, x.data(), out.data()), "multiply");
}

std::vector<double> SparseMatrix::multiply(std::span<const double> x) const {
  std::vector<double> out(static_cast<std::size_t>(num_rows_));
  multiply(x, out);
  return out;
}

void SparseMatrix::multiply_transpose(std::span<const double> y, std::span<double> out) const {
  if (static_cast<Index>(y.size()) != num_rows_ || static_cast<Index>(out.size()) != num_cols_) {
    throw DimensionMismatch("multiply_transpose: size mismatch");
  }
  if (num_cols_ == 0) return;
  device::Context ctx(*this);
  device::check(folp_gpu_multiply_transpose(ctx.get(), 0, y.data(), out.data()),
                "multiply_transpose");
}

std::vector<double> SparseMatrix::multiply_transpose(std::span<const double> y) const {
  std::vector<double> out(static_cast<std::size_t>(num_cols_));
  multiply_transpose(y, out);
  return out;
}

double SparseMatrix::max_abs_entry() const {
  if (nnz() == 0) throw EmptyMatrix("max_abs_entry: matrix has no entries");
  device::Context ctx(*this);
  double v = 0.0;
  device::check(folp_gpu_max_abs_entry(ctx.get(), 0, &v), "max_abs_entry");
  return v;
}

std::vector<double> SparseMatrix::axis_norms(Axis axis, double p) const {
  if (std::isnan(p) || (p < 1.0 && p != 0.0)) {
    throw UnsupportedNorm("axis_norms: p must be 0, in [1, inf), or +inf");
  }
  const bool rows = axis == Axis::kRows;
  std::vector<double> out(static_cast<std::size_t>(rows ? num_rows_ : num_cols_), 0.0);
  if (out.empty()) return out;
  device::Context ctx(*this);
  device::check(folp_gpu_axis_norms(ctx.get(), rows ? 0 : 1, p, 0, out.data()), "axis_norms");
  return out;
}

// estimate_spectral_norm (sparse_matrix.cpp:188-220): the start vector is
// drawn on the host from mt19937_64(seed) exactly like the reference
// (raw-draw U(-1,1), normalised); the power iteration runs on the device.
double SparseMatrix::estimate_spectral_norm(double relative_tol, Index max_iterations,
                                            std::uint64_t seed, Index* multiply_count) const {
  if (num_rows_ == 0 || num_cols_ == 0 || nnz() == 0) {
    throw EmptyMatrix("estimate_spectral_norm: empty matrix");
  }
  std::mt19937_64 rng(seed);
  std::vector<double> v(static_cast<std::size_t>(num_cols_));
  for (double& e : v) e = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
  double vnorm = linalg::norm2(v);
  if (vnorm == 0.0) {
    v[0] = 1.0;
    vnorm = 1.0;
  }
  linalg::scale(v, 1.0 / vnorm);
  device::Context ctx(*this);
  double norm = 0.0;
  int64_t count = 0;
  device::check(folp_gpu_spectral_norm(ctx.get(), v.data(), relative_tol, max_iterations, &norm,
                                       &count),
                "estimate_spectral_norm");
  if (multiply_count != nullptr) *multiply_count += count;
  return norm;
}

// scaled (sparse_matrix.cpp:222-242): a pure data transform of the stored
// values, kept on the host; the solve path scales on the device instead.
SparseMatrix SparseMatrix::scaled(std::span<const double> row_scale,
                                  std::span<const double> col_scale) const {
  if (static_cast<Index>(row_scale.size()) != num_rows_ ||
      static_cast<Index>(col_scale.size()) != num_cols_) {
    throw DimensionMismatch("scaled: scale vector size mismatch");
  }
  SparseMatrix out = *this;
  for (Index r = 0; r < num_rows_; ++r) {
    for (Index k = csr_start_[r]; k < csr_start_[r + 1]; ++k) {
      out.csr_values_[k] *= row_scale[r] * col_scale[csr_index_[k]];
    }
  }
  const ColumnMirror& cm = columns();
  auto mirror = std::make_shared<ColumnMirror>(cm);
  for (Index c = 0; c < num_cols_; ++c) {
    for (Index k = cm.start[c]; k < cm.start[c + 1]; ++k) {
      mirror->values[k] *= col_scale[c] * row_scale[cm.index[k]];
    }
  }
  out.csc_ = std::move(mirror);
  out.csc_mu_ = std::make_shared<std::mutex>();
  return out;
}

bool SparseMatrix::has_column_mirror() const {
  if (!csc_mu_) return csc_ != nullptr;  // moved-from
  std::lock_guard<std::mutex> lk(*csc_mu_);
  return csc_ != nullptr;
}

// The column-compressed mirror by a counting pass in row order: columns in
// increasing row order, the layout from_triplets produces
// (sparse_matrix.cpp:82-102).
const SparseMatrix::ColumnMirror& SparseMatrix::columns() const {
  if (!csc_mu_) csc_mu_ = std::make_shared<std::mutex>();  // moved-from, single owner
  std::lock_guard<std::mutex> lk(*csc_mu_);
  if (!csc_) {
    auto cm = std::make_shared<ColumnMirror>();
    const Index nnz = static_cast<Index>(csr_values_.size());
    cm->start.assign(static_cast<std::size_t>(num_cols_) + 1, 0);
    cm->index.resize(static_cast<std::size_t>(nnz));
    cm->values.resize(static_cast<std::size_t>(nnz));
    for (Index e = 0; e < nnz; ++e) ++cm->start[csr_index_[e] + 1];
    for (Index c = 0; c < num_cols_; ++c) cm->start[c + 1] += cm->start[c];
    std::vector<Index> fill(cm->start.begin(), cm->start.end() - 1);
    for (Index r = 0; r < num_rows_; ++r) {
      for (Index e = csr_start_[r]; e < csr_start_[r + 1]; ++e) {
        const Index slot = fill[csr_index_[e]]++;
        cm->index[slot] = r;
        cm->values[slot] = csr_values_[e];
      }
    }
    csc_ = std::move(cm);
  }
  return *csc_;
}

SparseMatrix SparseMatrixAccess::build(Index m, Index n, std::vector<Index> start,
                                       std::vector<Index> cols, std::vector<double> vals) {
  SparseMatrix k;
  k.num_rows_ = m;
  k.num_cols_ = n;
  k.csr_start_ = std::move(start);
  k.csr_index_ = std::move(cols);
  k.csr_values_ = std::move(vals);
  return k;  // column mirror on first use
}

SparseMatrix SparseMatrixAccess::with_values(const SparseMatrix& k, std::vector<double> csr,
                                             std::vector<double> csc) {
  SparseMatrix out;
  out.num_rows_ = k.num_rows_;
  out.num_cols_ = k.num_cols_;
  out.csr_start_ = k.csr_start_;
  out.csr_index_ = k.csr_index_;
  out.csr_values_ = std::move(csr);
  const SparseMatrix::ColumnMirror& cm = k.columns();
  auto mirror = std::make_shared<SparseMatrix::ColumnMirror>();
  mirror->start = cm.start;
  mirror->index = cm.index;
  mirror->values = std::move(csc);
  out.csc_ = std::move(mirror);
  return out;
}

}  // namespace folp
