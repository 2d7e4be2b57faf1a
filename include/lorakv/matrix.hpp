// lorakv/matrix.hpp -- boundary types of the operator API (Span2D, Matrix, fail, max_rel_error) and
// the dense matmul, source-compatible with proj/include/lorakv/matrix.hpp of the reference.
//
// The types are plain host containers: callers of the reference pass borrowed row-major views with
// an explicit row stride and receive owning matrices (matrix.hpp:31-38, 60-63).  Everything that
// COMPUTES goes to the B200 through the C ABI (include/lorakv_b200.h): matmul -> lorakv_matmul_*,
// whose accumulation order and roundings reproduce the reference's triple loop bit for bit
// (matrix.hpp:101-111 under -ffp-contract=off).  There is no host fallback: without the CUDA
// library and a B200 every operator throws std::runtime_error, the reference's only error type
// (matrix.hpp:17-19).  The host-only statistics of the reference (row_softmax, cosine, L1) belong
// to its analysis tools and are outside this path.
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "lorakv/rng.hpp"
#include "lorakv_b200.h"

namespace lorakv {

using idx = std::int64_t;

[[noreturn]] inline void fail(const std::string& msg) { throw std::runtime_error(msg); }

inline std::string shape_str(idx rows, idx cols) { return std::to_string(rows) + "x" + std::to_string(cols); }

// ---- the device behind the headers --------------------------------------------------------------
namespace b200 {

// One process-wide lorakv_ctx on device $LORAKV_B200_DEVICE (default 0), created on first use.
class Runtime {
 public:
  static lorakv_ctx* ctx() {
    static Runtime rt;
    return rt.ctx_;
  }
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

 private:
  Runtime() {
    const char* env = std::getenv("LORAKV_B200_DEVICE");
    if (lorakv_ctx_create(env ? std::atoi(env) : 0, nullptr, &ctx_) != LORAKV_OK) fail(lorakv_last_error());
  }
  ~Runtime() { lorakv_ctx_destroy(ctx_); }
  lorakv_ctx* ctx_ = nullptr;
};

inline void check(int status) {
  if (status != LORAKV_OK) fail(lorakv_last_error());
}

template <class T>
constexpr bool is_supported = std::is_same_v<T, float> || std::is_same_v<T, double>;

}  // namespace b200

// Borrowed view of row-major storage; `stride` counts elements between rows, so a column slice of a
// wider matrix (one attention head, attention.hpp:351-354) is a view, not a copy.
template <class T>
struct Span2D {
  const T* data = nullptr;
  idx rows = 0;
  idx cols = 0;
  idx stride = 0;

  const T* row(idx i) const { return data + i * stride; }
  const T& operator()(idx i, idx j) const { return row(i)[j]; }
  bool empty() const { return rows == 0 || cols == 0; }

  Span2D row_range(idx begin, idx end) const {
    if (begin < 0 || end < begin || end > rows) out_of_bounds("row_range", begin, end);
    return Span2D{data + begin * stride, end - begin, cols, stride};
  }
  Span2D col_range(idx begin, idx end) const {
    if (begin < 0 || end < begin || end > cols) out_of_bounds("col_range", begin, end);
    return Span2D{data + begin, rows, end - begin, stride};
  }

 private:
  [[noreturn]] void out_of_bounds(const char* what, idx begin, idx end) const {
    fail(std::string(what) + " [" + std::to_string(begin) + "," + std::to_string(end) + ") out of bounds for " +
         shape_str(rows, cols));
  }
};

// Owning dense row-major matrix.
template <class T>
struct Matrix {
  idx rows = 0;
  idx cols = 0;
  std::vector<T> data;

  Matrix() = default;
  Matrix(idx r, idx c) : rows(r), cols(c) {
    if (r < 0 || c < 0) fail("negative matrix shape " + shape_str(r, c));
    data.assign(static_cast<std::size_t>(r * c), T(0));
  }

  T& operator()(idx i, idx j) { return data[static_cast<std::size_t>(i * cols + j)]; }
  const T& operator()(idx i, idx j) const { return data[static_cast<std::size_t>(i * cols + j)]; }
  Span2D<const T> view() const { return Span2D<const T>{data.data(), rows, cols, cols}; }
  bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }

  static Matrix identity(idx n) {
    Matrix m(n, n);
    for (idx i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
  }
  // row-major fill, one gaussian draw per element, scaled in double then narrowed (matrix.hpp:83-87)
  static Matrix gaussian(idx r, idx c, Rng rng, double scale) {
    Matrix m(r, c);
    for (T& x : m.data) x = static_cast<T>(rng.gaussian() * scale);
    return m;
  }
};

template <class T>
inline void ensure_finite(const Matrix<T>& m, const char* op) {
  const bool ok = std::all_of(m.data.begin(), m.data.end(),
                              [](const T& v) { return std::isfinite(static_cast<double>(v)); });
  if (!ok) fail(std::string(op) + " produced a non-finite entry");
}

inline std::uint64_t matmul_macs(idx m, idx k, idx n) {
  return static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(k) * static_cast<std::uint64_t>(n);
}

// a (m x k) * b (k x n) on the device; bit-identical to the reference's i-p-j loop
template <class T>
inline Matrix<T> matmul(Span2D<const T> a, Span2D<const T> b) {
  static_assert(b200::is_supported<T>, "lorakv operators exist for float and double");
  if (a.cols != b.rows)
    fail("matmul dimension mismatch: " + shape_str(a.rows, a.cols) + " x " + shape_str(b.rows, b.cols));
  Matrix<T> out(a.rows, b.cols);
  if constexpr (std::is_same_v<T, float>)
    b200::check(lorakv_matmul_f32(b200::Runtime::ctx(), a.data, a.stride, b.data, b.stride, a.rows, a.cols, b.cols, out.data.data()));
  else
    b200::check(lorakv_matmul_f64(b200::Runtime::ctx(), a.data, a.stride, b.data, b.stride, a.rows, a.cols, b.cols, out.data.data()));
  return out;
}

template <class T>
inline Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b) {
  return matmul(a.view(), b.view());
}

// out += a * b (matrix.hpp:101-111).  The product runs on the device like matmul; into a zero `out` -- the only way the
// reference itself calls it (matmul, :114-121) -- the result carries the reference's bits, into anything else the product
// is added with one rounding per element instead of being threaded through the reference's running sum.
template <class T>
inline void matmul_accumulate(Span2D<const T> a, Span2D<const T> b, Matrix<T>& out) {
  if (a.cols != b.rows || out.rows != a.rows || out.cols != b.cols)
    fail("matmul dimension mismatch: " + shape_str(a.rows, a.cols) + " x " + shape_str(b.rows, b.cols));
  const Matrix<T> product = matmul(a, b);
  std::transform(out.data.begin(), out.data.end(), product.data.begin(), out.data.begin(), [](T x, T y) { return x + y; });
}

// ---- host statistics the reference's analysis tools and its naive oracle use (matrix.hpp:138-186).  Not on the device
// path: a few scalar passes over host matrices. ----

// softmax of every row after subtracting its maximum; -inf entries (masked scores) are fine, a row of nothing else is not
template <class T>
inline Matrix<T> row_softmax(const Matrix<T>& s) {
  const T ninf = -std::numeric_limits<T>::infinity();
  Matrix<T> out(s.rows, s.cols);
  for (idx i = 0; i < s.rows; ++i) {
    const T* in = s.data.data() + i * s.cols;
    T* o = out.data.data() + i * s.cols;
    const T top = s.cols > 0 ? *std::max_element(in, in + s.cols) : ninf;
    if (!(top > ninf)) fail("row_softmax: row " + std::to_string(i) + " has no finite entry");
    T total = T(0);
    for (idx j = 0; j < s.cols; ++j) total += (o[j] = std::exp(in[j] - top));
    for (idx j = 0; j < s.cols; ++j) o[j] /= total;
  }
  ensure_finite(out, "row_softmax");
  return out;
}

// cosine of the angle between two matrices seen as vectors, accumulated in double and clamped to [-1, 1]
template <class T>
inline double cosine_similarity(const Matrix<T>& a, const Matrix<T>& b) {
  if (!a.same_shape(b))
    fail("cosine_similarity shape mismatch: " + shape_str(a.rows, a.cols) + " vs " + shape_str(b.rows, b.cols));
  double ab = 0.0, aa = 0.0, bb = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    const double x = static_cast<double>(a.data[i]), y = static_cast<double>(b.data[i]);
    ab += x * y; aa += x * x; bb += y * y;
  }
  if (aa == 0.0 || bb == 0.0) fail("cosine_similarity: zero-norm input");
  return std::clamp(ab / (std::sqrt(aa) * std::sqrt(bb)), -1.0, 1.0);
}

// mean absolute entry (0 for an empty matrix)
template <class T>
inline double l1_norm_mean(const Matrix<T>& a) {
  if (a.data.empty()) return 0.0;
  double total = 0.0;
  for (const T& v : a.data) total += std::abs(static_cast<double>(v));
  return total / static_cast<double>(a.data.size());
}

template <class T>
inline Matrix<T> add(const Matrix<T>& a, const Matrix<T>& b) {
  if (!a.same_shape(b))
    fail("add shape mismatch: " + shape_str(a.rows, a.cols) + " vs " + shape_str(b.rows, b.cols));
  Matrix<T> out(a.rows, a.cols);
  std::transform(a.data.begin(), a.data.end(), b.data.begin(), out.data.begin(), [](T x, T y) { return x + y; });
  return out;
}

template <class T>
inline Matrix<T> scale(const Matrix<T>& a, T factor) {
  Matrix<T> out(a.rows, a.cols);
  std::transform(a.data.begin(), a.data.end(), out.data.begin(), [factor](T x) { return x * factor; });
  return out;
}

// THE parity metric (matrix.hpp:200-214): max |a - b| over the whole matrix, divided by max |b|
template <class T>
inline double max_rel_error(const Matrix<T>& a, const Matrix<T>& b) {
  if (!a.same_shape(b))
    fail("max_rel_error shape mismatch: " + shape_str(a.rows, a.cols) + " vs " + shape_str(b.rows, b.cols));
  double worst = 0.0, magnitude = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    const double x = static_cast<double>(a.data[i]), y = static_cast<double>(b.data[i]);
    worst = std::max(worst, std::abs(x - y));
    magnitude = std::max(magnitude, std::abs(y));
  }
  return worst == 0.0 ? 0.0 : worst / std::max(magnitude, 1e-300);
}

template <class T>
inline double max_abs_diff(const Matrix<T>& a, const Matrix<T>& b) {
  double worst = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i)
    worst = std::max(worst, std::abs(static_cast<double>(a.data[i]) - static_cast<double>(b.data[i])));
  return worst;
}

}  // namespace lorakv
