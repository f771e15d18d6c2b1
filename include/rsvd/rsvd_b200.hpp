// C++ drop-in for the reference's hot-path API (namespace rsvd), backed by the
// B200 engine through the C ABI in rsvd_b200.h.
//
// Mirrors /root/reference/proj/include/rsvd/:
//   core.hpp:18-66        DenseMatrix / Vector / Index, DimensionError,
//                         ParameterError, NumericError, SvdApprox, EvdApprox
//   core.hpp:96-177       orthonormalize, svd_small, evd_symmetric, solve_ls
//   core.hpp:180-221      singular_values, spectral_norm
//   bounds.hpp:107-120    computed_range_error
//   angles.hpp:11-78      AngleReport, canonical_sines, subspace_quality
//   sketch.hpp:19-59      Rng (std::mt19937_64 + std::normal_distribution), gaussian
//   rangefinder.hpp:13-105 RangeMode, SketchConfig, fixed_rank_range,
//                         power_range, subspace_iter_range, range_basis
//   factor.hpp:12-34      rsvd (both overloads), truncate
//   singlepass.hpp:15-137 CountingOperator, spevd_hermitian, spsvd_general
//
// DenseMatrix is Eigen::MatrixXd when Eigen is available (exactly the
// reference's type); otherwise a minimal column-major matrix with the same
// storage convention.  Every call takes host matrices, runs on the GPU (one
// engine handle per thread, device 0 unless rsvd::set_device is called) and
// returns owning host results, like the reference.  The Rng is the
// reference's own libstdc++ engine; the device advances its state exactly as
// the host draws would (its state is exported/imported through the standard
// stream operators of std::mt19937_64 / std::normal_distribution).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../rsvd_b200.h"

#if __has_include(<Eigen/Dense>) && !defined(RSVD_B200_NO_EIGEN)
#include <Eigen/Dense>
#define RSVD_B200_EIGEN 1
#endif

namespace rsvd {

#ifdef RSVD_B200_EIGEN
using DenseMatrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;

/// Minimal column-major fp64 matrix (the reference's storage convention).
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
  double& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), 0.0);
  }
  static DenseMatrix Zero(Index r, Index c) { return DenseMatrix(r, c); }
  static DenseMatrix Identity(Index r, Index c) {
    DenseMatrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  DenseMatrix transpose() const {
    DenseMatrix t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  DenseMatrix leftCols(Index k) const {
    DenseMatrix t(r_, k);
    std::copy(d_.begin(), d_.begin() + static_cast<std::ptrdiff_t>(r_ * k), t.d_.begin());
    return t;
  }
  DenseMatrix head(Index k) const { return leftCols(k).reshaped_vector(k); }
  bool allFinite() const {
    for (double v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  double maxAbs() const {
    double m = 0;
    for (double v : d_) m = std::max(m, std::abs(v));
    return m;
  }
  friend DenseMatrix operator*(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.c_ != b.r_) throw std::invalid_argument("DenseMatrix: inner dimensions differ");
    DenseMatrix c(a.r_, b.c_);
    for (Index j = 0; j < b.c_; ++j)
      for (Index k = 0; k < a.c_; ++k) {
        const double bk = b(k, j);
        for (Index i = 0; i < a.r_; ++i) c(i, j) += a(i, k) * bk;
      }
    return c;
  }
  friend DenseMatrix operator-(const DenseMatrix& a, const DenseMatrix& b) {
    DenseMatrix c = a;
    for (size_t i = 0; i < c.d_.size(); ++i) c.d_[i] -= b.d_[i];
    return c;
  }

 private:
  DenseMatrix reshaped_vector(Index k) const {
    DenseMatrix v(k, 1);
    std::copy(d_.begin(), d_.begin() + static_cast<std::ptrdiff_t>(k), v.d_.begin());
    return v;
  }
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};
using Vector = DenseMatrix;  // column vector (n x 1)
#endif

/// Bad shape (reference core.hpp:23-26).
class DimensionError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
/// Invalid parameter value (reference core.hpp:29-32).
class ParameterError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
/// Numerical failure (reference core.hpp:35-39).
class NumericError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace b200 {

inline int& device_slot() {
  thread_local int dev = 0;
  return dev;
}

struct HandleDeleter {
  void operator()(rsvd_handle* h) const { rsvd_destroy(h); }
};

[[noreturn]] inline void raise(rsvd_status st) {
  const std::string msg = rsvd_last_error();
  switch (st) {
    case RSVD_ERR_DIMENSION: throw DimensionError(msg);
    case RSVD_ERR_PARAMETER: throw ParameterError(msg);
    case RSVD_ERR_NUMERIC: throw NumericError(msg);
    default: throw std::runtime_error("rsvd-b200: " + msg);
  }
}
inline void check(rsvd_status st) {
  if (st != RSVD_OK) raise(st);
}

/// One engine handle per thread (lazily created on the selected device).
inline rsvd_handle* handle() {
  thread_local std::unique_ptr<rsvd_handle, HandleDeleter> h;
  thread_local int h_dev = -1;
  if (!h || h_dev != device_slot()) {
    rsvd_handle* raw = nullptr;
    check(rsvd_create(&raw, device_slot()));
    h.reset(raw);
    h_dev = device_slot();
  }
  return h.get();
}

}  // namespace b200

/// Select the GPU used by subsequent calls on this thread.
inline void set_device(int device) { b200::device_slot() = device; }

/// Factor triple U * diag(sigma) * V^T (reference core.hpp:43-53).
struct SvdApprox {
  DenseMatrix U;
  Vector sigma;
  DenseMatrix V;
  Index factor_count() const { return sigma.rows(); }
};

/// U * diag(lambda) * U^T, lambda ordered by |lambda| desc (core.hpp:57-66).
struct EvdApprox {
  DenseMatrix U;
  Vector lambda;
  Index factor_count() const { return lambda.rows(); }
};

// ------------------------------------------------------------- sketch.hpp
/// Seeded random stream, identical to the reference's (sketch.hpp:19-45).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  static constexpr std::string_view identity() { return "mt19937_64/std-normal/v1"; }
  double normal() { return normal_(engine_); }
  double uniform01() { return uniform_(engine_); }
  std::uint64_t index(std::uint64_t bound) {
    return std::uniform_int_distribution<std::uint64_t>(0, bound - 1)(engine_);
  }
  static Rng for_trial(std::uint64_t seed_base, std::uint64_t trial) {
    return Rng(seed_base + trial);
  }

  /// Export / import the full state for the device generator.
  rsvd_rng_state export_state() const {
    rsvd_rng_state st{};
    std::stringstream ss;
    ss << engine_;
    for (auto& w : st.mt) ss >> w;
    ss >> st.pos;
    std::stringstream ns;
    ns.precision(17);
    ns << normal_;
    double mean = 0, sd = 0;
    int avail = 0;
    ns >> mean >> sd >> avail;
    st.has_cached = avail;
    if (avail) ns >> st.cached;
    return st;
  }
  void import_state(const rsvd_rng_state& st) {
    std::stringstream ss;
    for (auto w : st.mt) ss << w << ' ';
    ss << st.pos;
    ss >> engine_;
    char buf[96];
    if (st.has_cached)
      std::snprintf(buf, sizeof buf, "0 1 1 %.17e", st.cached);
    else
      std::snprintf(buf, sizeof buf, "0 1 0");
    std::stringstream ds(buf);
    ds >> normal_;
  }

 private:
  std::mt19937_64 engine_;
  std::normal_distribution<double> normal_{0.0, 1.0};
  std::uniform_real_distribution<double> uniform_{0.0, 1.0};
};

}  // namespace rsvd

#include "rsvd_b200_impl.hpp"
