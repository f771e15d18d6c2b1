// Implementation half of rsvd_b200.hpp: the reference's hot-path functions,
// each a thin host wrapper over one C-ABI call (include/rsvd_b200.h).
#pragma once

namespace rsvd {

namespace b200 {
inline DenseMatrix make(Index r, Index c) {
  DenseMatrix m(r, c);
  return m;
}
inline Vector make_vec(Index n) {
#ifdef RSVD_B200_EIGEN
  return Vector(n);
#else
  return Vector(n, 1);
#endif
}
inline int64_t ld(const DenseMatrix& m) { return std::max<int64_t>(1, m.rows()); }
}  // namespace b200

/// n x l i.i.d. N(0,1), column-major (reference sketch.hpp:48-59).
inline DenseMatrix gaussian(Index n, Index l, Rng& rng) {
  if (n < 1 || l < 1) throw ParameterError("gaussian: dimensions must be positive");
  DenseMatrix m = b200::make(n, l);
  rsvd_rng_state st = rng.export_state();
  b200::check(rsvd_gaussian_host(b200::handle(), n, l, &st, m.data(), b200::ld(m)));
  rng.import_state(st);
  return m;
}

/// Householder-quality orthonormal basis, padded to full width
/// (reference core.hpp:96-105).
inline DenseMatrix orthonormalize(const DenseMatrix& m) {
  DenseMatrix q = b200::make(m.rows(), m.cols());
  b200::check(rsvd_orthonormalize_host(b200::handle(), m.rows(), m.cols(), m.data(), b200::ld(m),
                                       q.data(), b200::ld(q)));
  return q;
}

/// Thin SVD with the reference sign rule (core.hpp:111-124).
inline SvdApprox svd_small(const DenseMatrix& m) {
  const Index r = std::min(m.rows(), m.cols());
  SvdApprox f{b200::make(m.rows(), r), b200::make_vec(r), b200::make(m.cols(), r)};
  b200::check(rsvd_svd_small_host(b200::handle(), m.rows(), m.cols(), m.data(), b200::ld(m),
                                  f.U.data(), b200::ld(f.U), f.sigma.data(), f.V.data(),
                                  b200::ld(f.V)));
  return f;
}

/// Symmetric EVD, |lambda| descending (core.hpp:130-162).
inline EvdApprox evd_symmetric(const DenseMatrix& c) {
  if (c.rows() != c.cols()) throw DimensionError("evd_symmetric: matrix is not square");
  EvdApprox e{b200::make(c.rows(), c.rows()), b200::make_vec(c.rows())};
  b200::check(rsvd_evd_symmetric_host(b200::handle(), c.rows(), c.data(), b200::ld(c),
                                      e.U.data(), b200::ld(e.U), e.lambda.data()));
  return e;
}

/// Min-norm least squares, cutoff 1e-12 sigma_max (core.hpp:166-177).
inline DenseMatrix solve_ls(const DenseMatrix& g, const DenseMatrix& h) {
  if (g.rows() != h.rows())
    throw DimensionError("solve_ls: row counts differ (" + std::to_string(g.rows()) + " vs " +
                         std::to_string(h.rows()) + ")");
  DenseMatrix x = b200::make(g.cols(), h.cols());
  b200::check(rsvd_solve_ls_host(b200::handle(), g.rows(), g.cols(), g.data(), b200::ld(g),
                                 h.cols(), h.data(), b200::ld(h), x.data(), b200::ld(x)));
  return x;
}

// -------------------------------------------------------- rangefinder.hpp
enum class RangeMode { basic, power, power_ortho };

inline std::string_view to_string(RangeMode mode) {
  switch (mode) {
    case RangeMode::basic: return "basic";
    case RangeMode::power: return "power";
    case RangeMode::power_ortho: return "ortho";
  }
  return "?";
}

/// Every Stage-1 tunable (rangefinder.hpp:30-42).
struct SketchConfig {
  Index k = 1;
  Index p = 0;
  int q = 0;
  RangeMode mode = RangeMode::basic;
  std::uint64_t seed = 0;
  SketchConfig normalized() const {
    SketchConfig c = *this;
    if (c.mode == RangeMode::basic) c.q = 0;
    return c;
  }
};

inline DenseMatrix range_basis(const DenseMatrix& a, const SketchConfig& cfg, Rng& rng) {
  const SketchConfig c = cfg.normalized();
  DenseMatrix q = b200::make(a.rows(), std::max<Index>(c.k + c.p, 0));
  rsvd_rng_state st = rng.export_state();
  b200::check(rsvd_range_basis_host(b200::handle(), a.rows(), a.cols(), a.data(), b200::ld(a),
                                    c.k, c.p, c.q, static_cast<int>(c.mode), &st, q.data(),
                                    b200::ld(q)));
  rng.import_state(st);
  return q;
}
inline DenseMatrix fixed_rank_range(const DenseMatrix& a, Index k, Index p, Rng& rng) {
  return range_basis(a, SketchConfig{k, p, 0, RangeMode::basic, 0}, rng);
}
inline DenseMatrix power_range(const DenseMatrix& a, Index k, Index p, int q, Rng& rng) {
  return range_basis(a, SketchConfig{k, p, q, RangeMode::power, 0}, rng);
}
inline DenseMatrix subspace_iter_range(const DenseMatrix& a, Index k, Index p, int q, Rng& rng) {
  return range_basis(a, SketchConfig{k, p, q, RangeMode::power_ortho, 0}, rng);
}

// ------------------------------------------------------------- factor.hpp
/// Two-stage randomized SVD at full width k+p (factor.hpp:12-18).
inline SvdApprox rsvd(const DenseMatrix& a, const SketchConfig& cfg, Rng& rng) {
  const Index l = std::max<Index>(cfg.k + cfg.p, 0);
  SvdApprox f{b200::make(a.rows(), l), b200::make_vec(l), b200::make(a.cols(), l)};
  rsvd_rng_state st = rng.export_state();
  b200::check(rsvd_rsvd_host(b200::handle(), a.rows(), a.cols(), a.data(), b200::ld(a), cfg.k,
                             cfg.p, cfg.q, static_cast<int>(cfg.mode), &st, f.U.data(),
                             b200::ld(f.U), f.sigma.data(), f.V.data(), b200::ld(f.V)));
  rng.import_state(st);
  return f;
}
/// Convenience overload seeding the stream from cfg.seed (factor.hpp:21-24).
inline SvdApprox rsvd(const DenseMatrix& a, const SketchConfig& cfg) {
  Rng rng(cfg.seed);
  return rsvd(a, cfg, rng);
}
/// Keep the first k factor triples (factor.hpp:27-34).
inline SvdApprox truncate(const SvdApprox& f, Index k) {
  if (k < 0 || k > f.factor_count())
    throw DimensionError("truncate: k = " + std::to_string(k) + " exceeds factor count " +
                         std::to_string(f.factor_count()));
  SvdApprox t{b200::make(f.U.rows(), k), b200::make_vec(k), b200::make(f.V.rows(), k)};
  std::copy(f.U.data(), f.U.data() + f.U.rows() * k, t.U.data());
  std::copy(f.sigma.data(), f.sigma.data() + k, t.sigma.data());
  std::copy(f.V.data(), f.V.data() + f.V.rows() * k, t.V.data());
  return t;
}

// --------------------------------------------------------- singlepass.hpp
/// Operator view counting block applications (singlepass.hpp:15-40).  The
/// engine reports the applications it made; the counters are updated after
/// every single-pass call.
class CountingOperator {
 public:
  explicit CountingOperator(const DenseMatrix& a) : a_(&a) {}
  Index rows() const { return a_->rows(); }
  Index cols() const { return a_->cols(); }
  const DenseMatrix& matrix() const { return *a_; }
  int apply_count() const { return apply_count_; }
  int adjoint_count() const { return adjoint_count_; }
  void record(const rsvd_counters& before, const rsvd_counters& after) const {
    apply_count_ += static_cast<int>(after.apply - before.apply);
    adjoint_count_ += static_cast<int>(after.adjoint - before.adjoint);
  }

 private:
  const DenseMatrix* a_;
  mutable int apply_count_ = 0;
  mutable int adjoint_count_ = 0;
};

/// Single-pass symmetric EVD, Alg 5 (singlepass.hpp:45-73).
inline EvdApprox spevd_hermitian(const CountingOperator& op, Index k, Index p, Rng& rng) {
  const DenseMatrix& a = op.matrix();
  if (a.rows() != a.cols()) throw DimensionError("spevd_hermitian: matrix is not square");
  const Index kk = std::max<Index>(k, 0);
  EvdApprox e{b200::make(a.rows(), kk), b200::make_vec(kk)};
  rsvd_counters c0{}, c1{};
  rsvd_get_counters(b200::handle(), &c0);
  rsvd_rng_state st = rng.export_state();
  b200::check(rsvd_spevd_host(b200::handle(), a.rows(), a.data(), b200::ld(a), k, p, &st,
                              e.U.data(), b200::ld(e.U), e.lambda.data()));
  rng.import_state(st);
  rsvd_get_counters(b200::handle(), &c1);
  op.record(c0, c1);
  return e;
}
inline EvdApprox spevd_hermitian(const DenseMatrix& a, Index k, Index p, Rng& rng) {
  CountingOperator op(a);
  return spevd_hermitian(op, k, p, rng);
}

/// Single-pass general SVD, Alg 6 (singlepass.hpp:109-132).
inline SvdApprox spsvd_general(const CountingOperator& op, Index k, Index p, Rng& rng) {
  const DenseMatrix& a = op.matrix();
  const Index kk = std::max<Index>(k, 0);
  SvdApprox f{b200::make(a.rows(), kk), b200::make_vec(kk), b200::make(a.cols(), kk)};
  rsvd_counters c0{}, c1{};
  rsvd_get_counters(b200::handle(), &c0);
  rsvd_rng_state st = rng.export_state();
  b200::check(rsvd_spsvd_host(b200::handle(), a.rows(), a.cols(), a.data(), b200::ld(a), k, p,
                              &st, f.U.data(), b200::ld(f.U), f.sigma.data(), f.V.data(),
                              b200::ld(f.V)));
  rng.import_state(st);
  rsvd_get_counters(b200::handle(), &c1);
  op.record(c0, c1);
  return f;
}
inline SvdApprox spsvd_general(const DenseMatrix& a, Index k, Index p, Rng& rng) {
  CountingOperator op(a);
  return spsvd_general(op, k, p, rng);
}

// ------------------------------------- diagnostics (core / bounds / angles)
/// Singular values, descending (reference core.hpp:180-183).
inline Vector singular_values(const DenseMatrix& m) {
  const Index r = std::min(m.rows(), m.cols());
  Vector s = b200::make_vec(r);
  b200::check(rsvd_singular_values_host(b200::handle(), m.rows(), m.cols(), m.data(),
                                        b200::ld(m), s.data()));
  return s;
}

/// Largest singular value (reference core.hpp:188-221): dense SVD when
/// min(rows, cols) <= 512, else power iteration on M^T M (tol 1e-10, cap 5000).
inline double spectral_norm(const DenseMatrix& m) {
  double out = 0.0;
  b200::check(rsvd_spectral_norm_host(b200::handle(), m.rows(), m.cols(), m.data(), b200::ld(m),
                                      &out));
  return out;
}

/// Measured Stage-1 residual ||A - Q Q^T A||_2 (reference bounds.hpp:107-120).
inline double computed_range_error(const DenseMatrix& a, const DenseMatrix& q) {
  if (q.rows() != a.rows()) throw DimensionError("computed_range_error: row counts differ");
  double out = 0.0;
  b200::check(rsvd_computed_range_error_host(b200::handle(), a.rows(), a.cols(), a.data(),
                                             b200::ld(a), q.cols(), q.data(), b200::ld(q), &out));
  return out;
}

/// Per-index canonical-angle record (reference angles.hpp:11-22).
struct AngleReport {
  Index k = 0;
  Index p = 0;
  int q = 0;
  std::uint64_t seed = 0;
  double gap = 0.0;
  Vector sin_theta;
  Vector sin_nu;
  Vector bound_theta;
  Vector bound_nu;
};

/// Sines of the principal angles between range(X) and range(Y), ascending,
/// clamped to [0, 1] (reference angles.hpp:42-60, projection route).
inline Vector canonical_sines(const DenseMatrix& x, const DenseMatrix& y) {
  if (x.rows() != y.rows()) throw DimensionError("canonical_sines: ambient dimensions differ");
  Vector out = b200::make_vec(std::min(x.cols(), y.cols()));
  b200::check(rsvd_canonical_sines_host(b200::handle(), x.rows(), x.cols(), x.data(), b200::ld(x),
                                        y.cols(), y.data(), b200::ld(y), out.data()));
  return out;
}

/// Angles between the oracle's rank-k singular subspaces and the first k
/// computed factors (reference angles.hpp:62-78).
inline AngleReport subspace_quality(const SvdApprox& oracle, Index k, const SvdApprox& result) {
  if (k < 1) throw ParameterError("subspace_quality: k must be >= 1");
  if (oracle.factor_count() < k || result.factor_count() < k)
    throw DimensionError("subspace_quality: fewer than k factors available");
  AngleReport report;
  report.k = k;
  report.sin_theta = canonical_sines(oracle.U.leftCols(k), result.U.leftCols(k));
  report.sin_nu = canonical_sines(oracle.V.leftCols(k), result.V.leftCols(k));
  return report;
}
inline AngleReport subspace_quality(const DenseMatrix& a, Index k, const SvdApprox& result) {
  return subspace_quality(svd_small(a), k, result);
}

}  // namespace rsvd
