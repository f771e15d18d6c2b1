// ============================================================================
// rsvd CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A C++ restatement of the reference randomized-SVD hot path
// (/root/reference/proj/include/rsvd/{sketch,rangefinder,factor,singlepass,
// core}.hpp).  It exists to CHECK the B200 engine and to time the CPU
// baseline; only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
// reference arm may load it.  The product library (librsvd_b200.so) never
// links or calls anything in this directory.
//
// Fidelity:
//  * Omega stream: literally std::mt19937_64 + std::normal_distribution<double>
//    from the host libstdc++ — the same templates the reference instantiates
//    (sketch.hpp:19-45), filled column-major (sketch.hpp:48-59).
//  * Dense kernels: the reference calls Eigen (absent from this image, so the
//    reference cannot be compiled — see DESIGN.md).  Each Eigen call is
//    restated with the LAPACK routine implementing the same algorithm, taken
//    from scipy's bundled OpenBLAS 0.3.30:
//      Eigen GEMM                    -> dgemm
//      HouseholderQR + householderQ  -> dgeqrf + dorgqr (same beta = -sign(a)|x|)
//      BDCSVD (thin)                 -> dgesdd
//      SelfAdjointEigenSolver        -> dsyevd
//      BDCSVD::solve + threshold     -> dgesdd + explicit 1e-12 cutoff
//  * solve_joint_core (singlepass.hpp:84-101): the literal stacked
//    2l^2 x l^2 least-squares solve for l <= kStackedLimit, and the exactly
//    equivalent Kronecker-diagonalised O(l^3) solve above (the literal system
//    needs 1.46 TB at l = 550).  tests/ cross-check the two routes.
//
// Parity pin status: the reference ships no golden vectors.  The oracle is
// pinned by (a) the reference's own unit-test properties and known answers
// (tests/test_oracle_pins.py), and (b) the Omega stream being the reference's
// own libstdc++ generator (KAT: mt19937_64 10000th output, [rand.predef]).
// ============================================================================

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

extern "C" {
// scipy's bundled OpenBLAS (LP64, symbol prefix scipy_).
void scipy_dgemm_(const char*, const char*, const int*, const int*, const int*, const double*,
                  const double*, const int*, const double*, const int*, const double*, double*,
                  const int*, size_t, size_t);
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*, double*, const int*,
                   int*);
void scipy_dorgqr_(const int*, const int*, const int*, double*, const int*, const double*,
                   double*, const int*, int*);
void scipy_dgesdd_(const char*, const int*, const int*, double*, const int*, double*, double*,
                   const int*, double*, const int*, double*, const int*, int*, int*, size_t);
void scipy_dsyevd_(const char*, const char*, const int*, double*, const int*, double*, double*,
                   const int*, int*, const int*, int*, size_t, size_t);
void scipy_dgemv_(const char*, const int*, const int*, const double*, const double*, const int*,
                  const double*, const int*, const double*, double*, const int*, size_t);
void scipy_openblas_set_num_threads(int);
int scipy_openblas_get_num_threads(void);
}

namespace orc {

enum Status { kOk = 0, kDimension = 1, kParameter = 2, kNumeric = 3, kInternal = 9 };

struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParameterError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };

thread_local std::string g_last_error;

// Column-major dense matrix (the reference's storage convention, core.hpp:1-4).
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> d;
  const double* ext = nullptr;  // non-owning view (large read-only inputs: A)
  Mat() = default;
  Mat(int64_t rows, int64_t cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return d[static_cast<size_t>(i + j * r)]; }
  double operator()(int64_t i, int64_t j) const { return data()[static_cast<size_t>(i + j * r)]; }
  double* data() { return d.data(); }
  const double* data() const { return ext ? ext : d.data(); }
  static Mat from(int64_t rows, int64_t cols, const double* p) {
    Mat m(rows, cols);
    if (rows * cols > 0) std::memcpy(m.data(), p, sizeof(double) * rows * cols);
    return m;
  }
  static Mat view(int64_t rows, int64_t cols, const double* p) {
    Mat m;
    m.r = rows;
    m.c = cols;
    m.ext = p;
    return m;
  }
  void to(double* p) const {
    if (r * c > 0) std::memcpy(p, data(), sizeof(double) * r * c);
  }
  Mat transpose() const {
    Mat t(c, r);
    for (int64_t j = 0; j < c; ++j)
      for (int64_t i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  Mat left_cols(int64_t k) const {
    Mat t(r, k);
    if (r * k > 0) std::memcpy(t.data(), data(), sizeof(double) * r * k);
    return t;
  }
};

// C = op(A) * op(B)
Mat gemm(const Mat& a, bool ta, const Mat& b, bool tb) {
  const int64_t m = ta ? a.c : a.r, k = ta ? a.r : a.c;
  const int64_t kb = tb ? b.c : b.r, n = tb ? b.r : b.c;
  if (k != kb) throw DimensionError("gemm: inner dimensions differ");
  Mat c(m, n);
  if (m == 0 || n == 0) return c;
  if (k == 0) return c;
  const int mi = static_cast<int>(m), ni = static_cast<int>(n), ki = static_cast<int>(k);
  const int lda = static_cast<int>(std::max<int64_t>(1, a.r)), ldb = static_cast<int>(std::max<int64_t>(1, b.r));
  const double one = 1.0, zero = 0.0;
  scipy_dgemm_(ta ? "T" : "N", tb ? "T" : "N", &mi, &ni, &ki, &one, a.data(), &lda, b.data(), &ldb,
               &zero, c.data(), &mi, 1, 1);
  return c;
}

void require_finite(const Mat& m, const char* what) {
  const double* p = m.data();
  for (int64_t i = 0; i < m.r * m.c; ++i)
    if (!std::isfinite(p[i])) throw NumericError(std::string(what) + ": input has non-finite entries");
}

// ---------------------------------------------------------------- sketch.hpp
// Rng: reference sketch.hpp:19-45 — the SAME libstdc++ engine/distribution.
struct Rng {
  std::mt19937_64 engine;
  std::normal_distribution<double> normal{0.0, 1.0};
  explicit Rng(uint64_t seed) : engine(seed) {}
  double next_normal() { return normal(engine); }
};

// gaussian: reference sketch.hpp:48-59 (ParameterError :49-51, j outer / i inner :53-57).
Mat gaussian(int64_t n, int64_t l, Rng& rng) {
  if (n < 1 || l < 1) throw ParameterError("gaussian: dimensions must be positive");
  Mat m(n, l);
  for (int64_t j = 0; j < l; ++j)
    for (int64_t i = 0; i < n; ++i) m(i, j) = rng.next_normal();
  return m;
}

// ------------------------------------------------------------------ core.hpp
// orthonormalize: reference core.hpp:96-105 (Householder QR, thin Q).
Mat orthonormalize(const Mat& m) {
  if (m.c > m.r)
    throw DimensionError("orthonormalize: more columns than rows (" + std::to_string(m.c) + " > " +
                         std::to_string(m.r) + ")");
  require_finite(m, "orthonormalize");
  Mat q = m;
  const int mi = static_cast<int>(m.r), ni = static_cast<int>(m.c);
  if (ni == 0) return q;
  std::vector<double> tau(static_cast<size_t>(ni));
  int info = 0, lwork = -1;
  double wq = 0;
  scipy_dgeqrf_(&mi, &ni, q.data(), &mi, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgeqrf_(&mi, &ni, q.data(), &mi, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw NumericError("orthonormalize: dgeqrf failed");
  lwork = -1;
  scipy_dorgqr_(&mi, &ni, &ni, q.data(), &mi, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  work.assign(static_cast<size_t>(lwork), 0.0);
  scipy_dorgqr_(&mi, &ni, &ni, q.data(), &mi, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw NumericError("orthonormalize: dorgqr failed");
  return q;
}

struct Svd {
  Mat U;
  std::vector<double> s;
  Mat V;
};

// Thin SVD with dgesdd (the divide-and-conquer analogue of Eigen's BDCSVD).
Svd thin_svd(const Mat& m) {
  const int mi = static_cast<int>(m.r), ni = static_cast<int>(m.c);
  const int r = std::min(mi, ni);
  Svd out{Mat(m.r, r), std::vector<double>(static_cast<size_t>(r)), Mat(m.c, r)};
  if (r == 0) return out;
  Mat a = m;
  Mat vt(r, m.c);
  std::vector<int> iwork(static_cast<size_t>(8 * r));
  int info = 0, lwork = -1;
  double wq = 0;
  const int ldu = mi, ldvt = r;
  scipy_dgesdd_("S", &mi, &ni, a.data(), &mi, out.s.data(), out.U.data(), &ldu, vt.data(), &ldvt,
                &wq, &lwork, iwork.data(), &info, 1);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgesdd_("S", &mi, &ni, a.data(), &mi, out.s.data(), out.U.data(), &ldu, vt.data(), &ldvt,
                work.data(), &lwork, iwork.data(), &info, 1);
  if (info != 0) throw NumericError("svd: dgesdd did not converge");
  out.V = vt.transpose();
  return out;
}

// svd_small: reference core.hpp:111-124, including the sign rule (:115-122):
// the largest-|entry| of each U column (lowest row index on ties) is made
// nonnegative and the flip is propagated to V.
Svd svd_small(const Mat& m) {
  require_finite(m, "svd_small");
  Svd f = thin_svd(m);
  for (int64_t j = 0; j < f.U.c; ++j) {
    int64_t imax = 0;
    double best = -1.0;
    for (int64_t i = 0; i < f.U.r; ++i) {
      const double a = std::abs(f.U(i, j));
      if (a > best) { best = a; imax = i; }
    }
    if (f.U(imax, j) < 0.0) {
      for (int64_t i = 0; i < f.U.r; ++i) f.U(i, j) = -f.U(i, j);
      for (int64_t i = 0; i < f.V.r; ++i) f.V(i, j) = -f.V(i, j);
    }
  }
  return f;
}

struct Evd {
  Mat U;
  std::vector<double> lambda;
};

// evd_symmetric: reference core.hpp:130-162 (asymmetry check :135-140,
// symmetrize :141, eigensolve :142, stable sort by |lambda| desc :148-152).
Evd evd_symmetric(const Mat& c) {
  if (c.r != c.c) throw DimensionError("evd_symmetric: matrix is not square");
  require_finite(c, "evd_symmetric");
  const int64_t n = c.r;
  double maxabs = 0.0, asym = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      maxabs = std::max(maxabs, std::abs(c(i, j)));
      asym = std::max(asym, std::abs(c(i, j) - c(j, i)));
    }
  const double scale = 1.0 + maxabs;
  if (asym > 1e-8 * scale)
    throw NumericError("evd_symmetric: asymmetry " + std::to_string(asym) + " exceeds tolerance");
  Mat sym(n, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) sym(i, j) = 0.5 * (c(i, j) + c(j, i));
  std::vector<double> w(static_cast<size_t>(n));
  const int ni = static_cast<int>(n);
  int info = 0, lwork = -1, liwork = -1, iwq = 0;
  double wq = 0;
  if (n > 0) {
    scipy_dsyevd_("V", "L", &ni, sym.data(), &ni, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
    lwork = std::max(1, static_cast<int>(wq));
    liwork = std::max(1, iwq);
    std::vector<double> work(static_cast<size_t>(lwork));
    std::vector<int> iwork(static_cast<size_t>(liwork));
    scipy_dsyevd_("V", "L", &ni, sym.data(), &ni, w.data(), work.data(), &lwork, iwork.data(),
                  &liwork, &info, 1, 1);
    if (info != 0) throw NumericError("evd_symmetric: eigensolver failed");
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), int64_t{0});
  // Exact |lambda| ties go to the positive eigenvalue: Eigen returns the
  // spectrum of [[0,1],[1,0]] as (-1+d, 1), so the reference's stable |lambda|
  // sort yields (1, -1) (test_core.cpp:148-162); LAPACK returns exact +-1.
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    const double fa = std::abs(w[a]), fb = std::abs(w[b]);
    return fa != fb ? fa > fb : w[a] > w[b];
  });
  Evd out{Mat(n, n), std::vector<double>(static_cast<size_t>(n))};
  for (int64_t j = 0; j < n; ++j) {
    const int64_t src = order[static_cast<size_t>(j)];
    for (int64_t i = 0; i < n; ++i) out.U(i, j) = sym(i, src);
    out.lambda[static_cast<size_t>(j)] = w[static_cast<size_t>(src)];
  }
  return out;
}

constexpr double kLstsqRankCutoff = 1e-12;  // reference core.hpp:91

// solve_ls: reference core.hpp:166-177 — min-norm LS through a thin SVD,
// singular values < 1e-12 * sigma_max treated as zero.
Mat solve_ls(const Mat& g, const Mat& h) {
  if (g.r != h.r)
    throw DimensionError("solve_ls: row counts differ (" + std::to_string(g.r) + " vs " +
                         std::to_string(h.r) + ")");
  require_finite(g, "solve_ls");
  require_finite(h, "solve_ls");
  Svd f = thin_svd(g);
  const int64_t r = static_cast<int64_t>(f.s.size());
  const double thr = std::max(r ? f.s[0] * kLstsqRankCutoff : 0.0, std::numeric_limits<double>::min());
  int64_t rank = 0;
  while (rank < r && f.s[static_cast<size_t>(rank)] >= thr) ++rank;
  // x = V_r * diag(1/s_r) * U_r^T h
  Mat ur = f.U.left_cols(rank), vr = f.V.left_cols(rank);
  Mat t = gemm(ur, true, h, false);
  for (int64_t j = 0; j < t.c; ++j)
    for (int64_t i = 0; i < rank; ++i) t(i, j) /= f.s[static_cast<size_t>(i)];
  if (rank == 0) return Mat(g.c, h.c);
  return gemm(vr, false, t, false);
}

// --------------------------------------------------------- rangefinder.hpp
enum Mode { kBasic = 0, kPower = 1, kPowerOrtho = 2 };

// check_sketch_shape: reference rangefinder.hpp:46-55.
void check_sketch_shape(const Mat& a, int64_t k, int64_t p, int q) {
  if (k < 1) throw ParameterError("target rank k must be >= 1");
  if (p < 0) throw ParameterError("oversampling p must be >= 0");
  if (q < 0) throw ParameterError("power steps q must be >= 0");
  if (k + p > std::min(a.r, a.c))
    throw DimensionError("k+p = " + std::to_string(k + p) + " exceeds min(m,n) = " +
                         std::to_string(std::min(a.r, a.c)));
}

// fixed_rank_range: reference rangefinder.hpp:60-65 (Alg 2 Stage 1).
Mat fixed_rank_range(const Mat& a, int64_t k, int64_t p, Rng& rng) {
  check_sketch_shape(a, k, p, 0);
  const Mat omega = gaussian(a.c, k + p, rng);
  const Mat y = gemm(a, false, omega, false);
  return orthonormalize(y);
}

// power_range: reference rangefinder.hpp:70-79 (Alg 3, no re-orth).
Mat power_range(const Mat& a, int64_t k, int64_t p, int q, Rng& rng) {
  check_sketch_shape(a, k, p, q);
  const Mat omega = gaussian(a.c, k + p, rng);
  Mat y = gemm(a, false, omega, false);
  for (int j = 0; j < q; ++j) {
    const Mat z = gemm(a, true, y, false);
    y = gemm(a, false, z, false);
  }
  return orthonormalize(y);
}

// subspace_iter_range: reference rangefinder.hpp:83-94 (Alg 4).
Mat subspace_iter_range(const Mat& a, int64_t k, int64_t p, int q, Rng& rng) {
  check_sketch_shape(a, k, p, q);
  const Mat omega = gaussian(a.c, k + p, rng);
  const Mat y = gemm(a, false, omega, false);
  Mat qm = orthonormalize(y);
  for (int j = 0; j < q; ++j) {
    const Mat w = orthonormalize(gemm(a, true, qm, false));
    qm = orthonormalize(gemm(a, false, w, false));
  }
  return qm;
}

// range_basis: reference rangefinder.hpp:97-105 (+ normalized() :37-41).
Mat range_basis(const Mat& a, int64_t k, int64_t p, int q, int mode, Rng& rng) {
  if (mode == kBasic) q = 0;
  switch (mode) {
    case kBasic: return fixed_rank_range(a, k, p, rng);
    case kPower: return power_range(a, k, p, q, rng);
    case kPowerOrtho: return subspace_iter_range(a, k, p, q, rng);
  }
  throw ParameterError("unknown range mode");
}

// -------------------------------------------------------------- factor.hpp
// rsvd: reference factor.hpp:12-18 — B = Q^T A, svd_small(B), U = Q U_B.
Svd rsvd(const Mat& a, int64_t k, int64_t p, int q, int mode, Rng& rng) {
  const Mat qm = range_basis(a, k, p, q, mode, rng);
  const Mat b = gemm(qm, true, a, false);
  Svd f = svd_small(b);
  f.U = gemm(qm, false, f.U, false);
  return f;
}

// ---------------------------------------------------------- singlepass.hpp
// spevd_hermitian: reference singlepass.hpp:45-73 (Alg 5).
Evd spevd_hermitian(const Mat& a, int64_t k, int64_t p, Rng& rng, int* applies) {
  if (a.r != a.c) throw DimensionError("spevd_hermitian: matrix is not square");
  double maxabs = 0.0, asym = 0.0;
  for (int64_t j = 0; j < a.c; ++j)
    for (int64_t i = 0; i < a.r; ++i) {
      maxabs = std::max(maxabs, std::abs(a(i, j)));
      asym = std::max(asym, std::abs(a(i, j) - a(j, i)));
    }
  if (asym > 1e-8 * (1.0 + maxabs)) throw NumericError("spevd_hermitian: input is not symmetric");
  if (k < 1) throw ParameterError("spevd_hermitian: k must be >= 1");
  if (p < 0) throw ParameterError("spevd_hermitian: p must be >= 0");
  if (k + p > a.r) throw DimensionError("spevd_hermitian: k+p exceeds n");
  const int64_t n = a.r;
  const Mat omega = gaussian(n, k + p, rng);
  const Mat y = gemm(a, false, omega, false);  // the single pass over A
  if (applies) ++*applies;
  const Mat q = orthonormalize(y);
  const Mat g = gemm(q, true, omega, false);
  const Mat h = gemm(q, true, y, false);
  Mat c = solve_ls(g.transpose(), h.transpose()).transpose();
  Mat cs(c.r, c.c);
  for (int64_t j = 0; j < c.c; ++j)
    for (int64_t i = 0; i < c.r; ++i) cs(i, j) = 0.5 * (c(i, j) + c(j, i));
  Evd e = evd_symmetric(cs);
  Evd out{gemm(q, false, e.U.left_cols(k), false),
          std::vector<double>(e.lambda.begin(), e.lambda.begin() + k)};
  return out;
}

constexpr int64_t kStackedLimit = 40;

// solve_joint_core, literal route: reference singlepass.hpp:84-101.
Mat solve_joint_core_stacked(const Mat& g1, const Mat& h1, const Mat& g2, const Mat& h2) {
  const int64_t l = g1.r;
  Mat stacked(2 * l * l, l * l);
  Mat rhs(2 * l * l, 1);
  for (int64_t c = 0; c < l; ++c) {
    for (int64_t j = 0; j < l; ++j)
      for (int64_t i = 0; i < l; ++i) stacked(c * l + i, c * l + j) = g1(i, j);
    for (int64_t i = 0; i < l; ++i) rhs(c * l + i, 0) = h1(i, c);
  }
  for (int64_t c = 0; c < l; ++c) {
    for (int64_t j = 0; j < l; ++j)
      for (int64_t i = 0; i < l; ++i) stacked(l * l + c * l + i, j * l + i) = g2(j, c);
    for (int64_t i = 0; i < l; ++i) rhs(l * l + c * l + i, 0) = h2(i, c);
  }
  const Mat vec_c = solve_ls(stacked, rhs);
  return Mat::from(l, l, vec_c.data());
}

// solve_joint_core, Kronecker route (exactly the min-norm solution of the
// same stacked system): G1 = U1 S1 V1^T, G2 = U2 S2 V2^T, C = V1 X U2^T with
// X_ij = (s1_i a_ij + s2_j b_ij) / (s1_i^2 + s2_j^2), a = U1^T H1 U2,
// b = V1^T H2 V2; the stacked singular values are sqrt(s1_i^2 + s2_j^2) and
// the 1e-12 cutoff of solve_ls applies to them.
Mat solve_joint_core_kron(const Mat& g1, const Mat& h1, const Mat& g2, const Mat& h2) {
  const int64_t l = g1.r;
  if (g1.c != l || g2.r != l || g2.c != l || h1.r != l || h1.c != l || h2.r != l || h2.c != l)
    throw DimensionError("solve_joint_core: blocks must be l x l");
  require_finite(g1, "solve_ls");
  require_finite(h1, "solve_ls");
  require_finite(g2, "solve_ls");
  require_finite(h2, "solve_ls");
  Svd f1 = thin_svd(g1), f2 = thin_svd(g2);
  const Mat a = gemm(gemm(f1.U, true, h1, false), false, f2.U, false);
  const Mat b = gemm(gemm(f1.V, true, h2, false), false, f2.V, false);
  const double smax = std::sqrt(f1.s[0] * f1.s[0] + f2.s[0] * f2.s[0]);
  const double thr = std::max(smax * kLstsqRankCutoff, std::numeric_limits<double>::min());
  Mat x(l, l);
  for (int64_t j = 0; j < l; ++j)
    for (int64_t i = 0; i < l; ++i) {
      const double s1 = f1.s[static_cast<size_t>(i)], s2 = f2.s[static_cast<size_t>(j)];
      const double den = s1 * s1 + s2 * s2;
      if (std::sqrt(den) < thr) continue;
      x(i, j) = (s1 * a(i, j) + s2 * b(i, j)) / den;
    }
  return gemm(gemm(f1.V, false, x, false), false, f2.U, true);
}

Mat solve_joint_core(const Mat& g1, const Mat& h1, const Mat& g2, const Mat& h2) {
  return g1.r <= kStackedLimit ? solve_joint_core_stacked(g1, h1, g2, h2)
                               : solve_joint_core_kron(g1, h1, g2, h2);
}

// spsvd_general: reference singlepass.hpp:109-132 (Alg 6).
Svd spsvd_general(const Mat& a, int64_t k, int64_t p, Rng& rng, int* applies, int* adjoints) {
  if (k < 1) throw ParameterError("spsvd_general: k must be >= 1");
  if (p < 0) throw ParameterError("spsvd_general: p must be >= 0");
  if (k + p > std::min(a.r, a.c)) throw DimensionError("spsvd_general: k+p exceeds min(m,n)");
  const int64_t m = a.r, n = a.c, l = k + p;
  const Mat omega_c = gaussian(n, l, rng);
  const Mat omega_r = gaussian(m, l, rng);
  const Mat y_c = gemm(a, false, omega_c, false);
  if (applies) ++*applies;
  const Mat y_r = gemm(a, true, omega_r, false);
  if (adjoints) ++*adjoints;
  const Mat q_c = orthonormalize(y_c);
  const Mat q_r = orthonormalize(y_r);
  const Mat c = solve_joint_core(gemm(omega_r, true, q_c, false), gemm(y_r, true, q_r, false),
                                 gemm(q_r, true, omega_c, false), gemm(q_c, true, y_c, false));
  Svd f = svd_small(c);
  Svd out{gemm(q_c, false, f.U.left_cols(k), false),
          std::vector<double>(f.s.begin(), f.s.begin() + k),
          gemm(q_r, false, f.V.left_cols(k), false)};
  return out;
}

// ------------------------------------------------- diagnostics (§8(f) rows 1, 3)
// singular_values: reference core.hpp:180-183 (dense_singular_values :77-79,
// BDCSVD values only -> dgesdd jobz = 'N').
std::vector<double> singular_values(const Mat& m) {
  require_finite(m, "singular_values");
  const int mi = static_cast<int>(m.r), ni = static_cast<int>(m.c);
  const int r = std::min(mi, ni);
  std::vector<double> s(static_cast<size_t>(std::max(r, 0)));
  if (r == 0) return s;
  Mat a = Mat::from(m.r, m.c, m.data());
  std::vector<int> iwork(static_cast<size_t>(8 * r));
  int info = 0, lwork = -1, one = 1;
  double wq = 0, dummy = 0;
  scipy_dgesdd_("N", &mi, &ni, a.data(), &mi, s.data(), &dummy, &one, &dummy, &one, &wq, &lwork,
                iwork.data(), &info, 1);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgesdd_("N", &mi, &ni, a.data(), &mi, s.data(), &dummy, &one, &dummy, &one, work.data(),
                &lwork, iwork.data(), &info, 1);
  if (info != 0) throw NumericError("singular_values: dgesdd did not converge");
  return s;
}

// Eigen's Vector::norm(): sqrt of the plain sum of squares.
double vnorm(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

// spectral_norm: reference core.hpp:188-221, statement by statement (dense
// route for min <= 512; LCG start vector; power iteration on M^T M with
// |est - sigma| <= 1e-10 est; NumericError after 5000 steps).
double spectral_norm(const Mat& m, int* iterations) {
  require_finite(m, "spectral_norm");
  if (iterations) *iterations = 0;
  if (std::min(m.r, m.c) <= 512) {
    std::vector<double> s = singular_values(m);
    return s.empty() ? 0.0 : s[0];
  }
  std::vector<double> x(static_cast<size_t>(m.c)), y(static_cast<size_t>(m.r));
  std::uint64_t state = 0x9e3779b97f4a7c15ULL;
  for (auto& xi : x) {
    state = state * 6364136223846793005ULL + 1442695040888963407ULL;
    xi = static_cast<double>(state >> 11) / 9007199254740992.0 - 0.5;
  }
  const double xn = vnorm(x);
  if (xn == 0.0) return 0.0;
  for (auto& xi : x) xi /= xn;
  const int mi = static_cast<int>(m.r), ni = static_cast<int>(m.c), inc = 1;
  const double one = 1.0, zero = 0.0;
  double sigma = 0.0;
  for (int iter = 0; iter < 5000; ++iter) {
    if (iterations) *iterations = iter + 1;
    scipy_dgemv_("N", &mi, &ni, &one, m.data(), &mi, x.data(), &inc, &zero, y.data(), &inc, 1);
    const double estimate = vnorm(y);
    if (estimate == 0.0) return 0.0;
    if (iter > 0 && std::abs(estimate - sigma) <= 1e-10 * estimate) return estimate;
    sigma = estimate;
    scipy_dgemv_("T", &mi, &ni, &one, m.data(), &mi, y.data(), &inc, &zero, x.data(), &inc, 1);
    const double nx = vnorm(x);
    if (nx == 0.0) return estimate;
    for (auto& xi : x) xi /= nx;
  }
  throw NumericError("spectral_norm: power iteration hit the 5000-step cap");
}

// max |X^T X - I| (reference angles.hpp:24-35, bounds.hpp:111-117)
double orthonormal_deviation(const Mat& x) {
  const Mat g = gemm(x, true, x, false);
  double dev = 0.0;
  for (int64_t j = 0; j < g.c; ++j)
    for (int64_t i = 0; i < g.r; ++i) dev = std::max(dev, std::abs(g(i, j) - (i == j ? 1.0 : 0.0)));
  return dev;
}

// computed_range_error: reference bounds.hpp:107-120.
double computed_range_error(const Mat& a, const Mat& q) {
  if (q.r != a.r) throw DimensionError("computed_range_error: row counts differ");
  const double dev = orthonormal_deviation(q);
  if (dev > 1e-8)
    throw NumericError("computed_range_error: Q is not orthonormal (deviation " +
                       std::to_string(dev) + ")");
  Mat resid = Mat::from(a.r, a.c, a.data());
  if (q.c > 0) {
    const Mat qa = gemm(q, true, a, false);
    const Mat qqa = gemm(q, false, qa, false);
    for (size_t i = 0; i < resid.d.size(); ++i) resid.d[i] -= qqa.d[i];
  }
  return spectral_norm(resid, nullptr);
}

// canonical_sines: reference angles.hpp:42-60 (projection route).
std::vector<double> canonical_sines(const Mat& x, const Mat& y) {
  if (x.r != y.r) throw DimensionError("canonical_sines: ambient dimensions differ");
  for (int w = 0; w < 2; ++w) {
    const double dev = orthonormal_deviation(w ? y : x);
    if (dev > 1e-8)
      throw NumericError(std::string("canonical_sines: ") + (w ? "Y" : "X") +
                         ": columns are not orthonormal (deviation " + std::to_string(dev) + ")");
  }
  Mat resid = Mat::from(y.r, y.c, y.data());
  if (x.c > 0) {
    const Mat xy = gemm(x, true, y, false);
    const Mat xxy = gemm(x, false, xy, false);
    for (size_t i = 0; i < resid.d.size(); ++i) resid.d[i] -= xxy.d[i];
  }
  const std::vector<double> sv = singular_values(resid);
  const int64_t count = std::min(x.c, y.c);
  std::vector<double> out(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i)
    out[static_cast<size_t>(i)] = std::clamp(sv[static_cast<size_t>(count - 1 - i)], 0.0, 1.0);
  return out;
}

// The RNG state exchanged with the engine (same layout as include/rsvd_b200.h).
struct RngState {
  uint64_t mt[312];
  uint64_t pos;
  int32_t has_cached;
  int32_t pad;
  double cached;
};

void get_state(const Rng& rng, RngState* st) {
  std::ostringstream os;
  os << rng.engine;
  std::istringstream is(os.str());
  for (int i = 0; i < 312; ++i) is >> st->mt[i];
  is >> st->pos;
  // normal_distribution serialization: mean stddev saved_available [saved]
  std::ostringstream ns;
  ns.precision(17);
  ns << rng.normal;
  std::istringstream nis(ns.str());
  double mean, sd;
  int avail = 0;
  nis >> mean >> sd >> avail;
  st->has_cached = avail;
  st->pad = 0;
  st->cached = 0.0;
  if (avail) nis >> st->cached;
}

void set_state(Rng& rng, const RngState* st) {
  std::ostringstream os;
  for (int i = 0; i < 312; ++i) os << st->mt[i] << ' ';
  os << st->pos;
  std::istringstream is(os.str());
  is >> rng.engine;
  // normal_distribution stream format: mean stddev saved_available [saved];
  // %.17e round-trips a double exactly.
  char buf[96];
  if (st->has_cached)
    std::snprintf(buf, sizeof buf, "0 1 1 %.17e", st->cached);
  else
    std::snprintf(buf, sizeof buf, "0 1 0");
  std::istringstream ds(buf);
  ds >> rng.normal;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const DimensionError& e) {
    g_last_error = e.what();
    return kDimension;
  } catch (const ParameterError& e) {
    g_last_error = e.what();
    return kParameter;
  } catch (const NumericError& e) {
    g_last_error = e.what();
    return kNumeric;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kInternal;
  }
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* orc_last_error() { return g_last_error.c_str(); }
void orc_set_threads(int n) { scipy_openblas_set_num_threads(n); }
// The compiler that instantiated the libstdc++ <random> templates of the Omega stream.
const char* orc_compiler() { return "g++ " __VERSION__; }
int orc_get_threads() { return scipy_openblas_get_num_threads(); }

void* orc_rng_new(uint64_t seed) { return new Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
double orc_rng_normal(void* r) { return static_cast<Rng*>(r)->next_normal(); }
uint64_t orc_rng_raw(void* r) { return static_cast<Rng*>(r)->engine(); }

// The accepted polar inputs r2 of the next `count` accepted attempts of the
// reference stream (libstdc++ random.tcc:1827-1834: x, y = 2u - 1 from
// generate_canonical; reject r2 > 1 or r2 == 0), and glibc's log of each.
void orc_polar_r2_log(void* r, int64_t count, double* r2_out, double* log_out) {
  auto& g = static_cast<Rng*>(r)->engine;
  for (int64_t i = 0; i < count;) {
    const double x = 2.0 * std::generate_canonical<double, 53>(g) - 1.0;
    const double y = 2.0 * std::generate_canonical<double, 53>(g) - 1.0;
    const double r2 = x * x + y * y;
    if (r2 > 1.0 || r2 == 0.0) continue;
    r2_out[i] = r2;
    log_out[i] = std::log(r2);
    ++i;
  }
}
void orc_rng_get_state(void* r, RngState* st) { get_state(*static_cast<Rng*>(r), st); }
void orc_rng_set_state(void* r, const RngState* st) { set_state(*static_cast<Rng*>(r), st); }

int orc_gaussian(int64_t n, int64_t l, void* rng, double* out) {
  return guard([&] { gaussian(n, l, *static_cast<Rng*>(rng)).to(out); });
}

int orc_gemm(int64_t m, int64_t n, int64_t k, const double* a, int ta, const double* b, int tb,
             double* c) {
  return guard([&] {
    Mat am = ta ? Mat::from(k, m, a) : Mat::from(m, k, a);
    Mat bm = tb ? Mat::from(n, k, b) : Mat::from(k, n, b);
    gemm(am, ta, bm, tb).to(c);
  });
}

int orc_orthonormalize(int64_t m, int64_t n, const double* a, double* q) {
  return guard([&] { orthonormalize(Mat::from(m, n, a)).to(q); });
}

int orc_svd_small(int64_t m, int64_t n, const double* a, double* u, double* s, double* v) {
  return guard([&] {
    Svd f = svd_small(Mat::from(m, n, a));
    f.U.to(u);
    std::copy(f.s.begin(), f.s.end(), s);
    f.V.to(v);
  });
}

int orc_evd_symmetric(int64_t n, const double* c, double* u, double* lambda) {
  return guard([&] {
    Evd e = evd_symmetric(Mat::from(n, n, c));
    e.U.to(u);
    std::copy(e.lambda.begin(), e.lambda.end(), lambda);
  });
}

int orc_solve_ls(int64_t m, int64_t n, const double* g, int64_t nrhs, const double* h, double* x) {
  return guard([&] { solve_ls(Mat::from(m, n, g), Mat::from(m, nrhs, h)).to(x); });
}

int orc_range_basis(int64_t m, int64_t n, const double* a, int64_t k, int64_t p, int q, int mode,
                    void* rng, double* qout) {
  return guard(
      [&] { range_basis(Mat::view(m, n, a), k, p, q, mode, *static_cast<Rng*>(rng)).to(qout); });
}

int orc_rsvd(int64_t m, int64_t n, const double* a, int64_t k, int64_t p, int q, int mode,
             void* rng, double* u, double* s, double* v) {
  return guard([&] {
    Svd f = rsvd(Mat::view(m, n, a), k, p, q, mode, *static_cast<Rng*>(rng));
    f.U.to(u);
    std::copy(f.s.begin(), f.s.end(), s);
    f.V.to(v);
  });
}

int orc_spevd(int64_t n, const double* a, int64_t k, int64_t p, void* rng, double* u,
              double* lambda, int* applies) {
  return guard([&] {
    Evd e = spevd_hermitian(Mat::view(n, n, a), k, p, *static_cast<Rng*>(rng), applies);
    e.U.to(u);
    std::copy(e.lambda.begin(), e.lambda.end(), lambda);
  });
}

int orc_spsvd(int64_t m, int64_t n, const double* a, int64_t k, int64_t p, void* rng, double* u,
              double* s, double* v, int* applies, int* adjoints) {
  return guard([&] {
    Svd f = spsvd_general(Mat::view(m, n, a), k, p, *static_cast<Rng*>(rng), applies, adjoints);
    f.U.to(u);
    std::copy(f.s.begin(), f.s.end(), s);
    f.V.to(v);
  });
}

int orc_solve_joint_core(int64_t l, const double* g1, const double* h1, const double* g2,
                         const double* h2, int route, double* c) {
  return guard([&] {
    Mat G1 = Mat::from(l, l, g1), H1 = Mat::from(l, l, h1), G2 = Mat::from(l, l, g2),
        H2 = Mat::from(l, l, h2);
    Mat r = route == 0   ? solve_joint_core_stacked(G1, H1, G2, H2)
            : route == 1 ? solve_joint_core_kron(G1, H1, G2, H2)
                         : solve_joint_core(G1, H1, G2, H2);
    r.to(c);
  });
}

int orc_singular_values(int64_t m, int64_t n, const double* a, double* s) {
  return guard([&] {
    const std::vector<double> v = singular_values(Mat::view(m, n, a));
    std::copy(v.begin(), v.end(), s);
  });
}

int orc_spectral_norm(int64_t m, int64_t n, const double* a, double* out, int* iterations) {
  return guard([&] { *out = spectral_norm(Mat::view(m, n, a), iterations); });
}

int orc_computed_range_error(int64_t m, int64_t n, const double* a, int64_t l, const double* q,
                             double* out) {
  return guard([&] { *out = computed_range_error(Mat::view(m, n, a), Mat::view(m, l, q)); });
}

int orc_canonical_sines(int64_t m, int64_t kx, const double* x, int64_t ky, const double* y,
                        double* out) {
  return guard([&] {
    const std::vector<double> v = canonical_sines(Mat::view(m, kx, x), Mat::view(m, ky, y));
    std::copy(v.begin(), v.end(), out);
  });
}

}  // extern "C"
