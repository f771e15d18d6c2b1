// C++ drop-in check: reference unit tests (proj/tests/unit/test_*.cpp) written
// against the same API, compiled against include/rsvd/ and linked to the B200
// engine.  Catch2 is absent from the image, so a minimal REQUIRE is used.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "rsvd/angles.hpp"
#include "rsvd/bounds.hpp"
#include "rsvd/factor.hpp"
#include "rsvd/singlepass.hpp"

static int g_fail = 0;
#define REQUIRE(x)                                                       \
  do {                                                                   \
    if (!(x)) {                                                          \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #x);         \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)
#define REQUIRE_THROWS_AS(expr, T) \
  do {                             \
    bool ok_ = false;              \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      ok_ = true;                  \
    }                              \
    REQUIRE(ok_);                  \
  } while (0)

using rsvd::DenseMatrix;
using rsvd::Rng;

static DenseMatrix random_matrix(rsvd::Index r, rsvd::Index c, std::uint64_t seed) {
  std::mt19937_64 eng(seed);
  std::normal_distribution<double> nd;
  DenseMatrix m(r, c);
  for (rsvd::Index j = 0; j < c; ++j)
    for (rsvd::Index i = 0; i < r; ++i) m(i, j) = nd(eng);
  return m;
}

static double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b) {
  double m = 0;
  for (rsvd::Index j = 0; j < a.cols(); ++j)
    for (rsvd::Index i = 0; i < a.rows(); ++i) m = std::max(m, std::abs(a(i, j) - b(i, j)));
  return m;
}

int main() {
  // test_sketch.cpp:11-20 and oracles.hpp:56-64: the device stream equals the
  // host libstdc++ stream (bit-exact except where glibc log is not CR).
  {
    Rng r1(42), r2(42);
    const DenseMatrix a = rsvd::gaussian(5, 3, r1);
    const DenseMatrix b = rsvd::gaussian(5, 3, r2);
    REQUIRE(max_abs_diff(a, b) == 0.0);
    const DenseMatrix ref = random_matrix(5, 3, 42);
    REQUIRE(max_abs_diff(a, ref) <= 1e-15);
    // the Rng continues exactly where the host library would
    Rng host(42);
    for (int i = 0; i < 15; ++i) host.normal();
    REQUIRE(r1.normal() == host.normal());
    REQUIRE(Rng::identity() == "mt19937_64/std-normal/v1");
  }
  // test_core.cpp:28-36
  {
    DenseMatrix m(3, 1);
    m(0, 0) = 3.0;
    m(1, 0) = 0.0;
    m(2, 0) = 4.0;
    const DenseMatrix q = rsvd::orthonormalize(m);
    const double sign = q(0, 0) > 0 ? 1.0 : -1.0;
    REQUIRE(std::abs(sign * q(0, 0) - 0.6) < 1e-12 && std::abs(sign * q(2, 0) - 0.8) < 1e-12);
    REQUIRE_THROWS_AS(rsvd::orthonormalize(DenseMatrix::Identity(2, 4)), rsvd::DimensionError);
  }
  // test_core.cpp:76-84
  {
    DenseMatrix m = DenseMatrix::Zero(3, 3);
    m(0, 0) = 3.0;
    m(1, 1) = 2.0;
    m(2, 2) = 1.0;
    const rsvd::SvdApprox f = rsvd::svd_small(m);
    REQUIRE(std::abs(f.sigma(0) - 3.0) < 1e-12);
    REQUIRE(std::abs(f.sigma(1) - 2.0) < 1e-12);
    REQUIRE(std::abs(f.sigma(2) - 1.0) < 1e-12);
  }
  // test_core.cpp:148-162
  {
    DenseMatrix c(2, 2);
    c(0, 0) = 0.0;
    c(0, 1) = 1.0;
    c(1, 0) = 1.0;
    c(1, 1) = 0.0;
    const rsvd::EvdApprox e = rsvd::evd_symmetric(c);
    REQUIRE(std::abs(e.lambda(0) - 1.0) < 1e-12);
    REQUIRE(std::abs(e.lambda(1) + 1.0) < 1e-12);
  }
  // test_factor.cpp:13-22 and :73-83
  {
    DenseMatrix a = DenseMatrix::Zero(3, 3);
    a(0, 0) = 3.0;
    a(1, 1) = 2.0;
    a(2, 2) = 1.0;
    const rsvd::SvdApprox f = rsvd::rsvd(a, rsvd::SketchConfig{3, 0, 0, rsvd::RangeMode::basic, 1});
    REQUIRE(std::abs(f.sigma(0) - 3.0) < 1e-10);
    REQUIRE(std::abs(f.sigma(2) - 1.0) < 1e-10);
    const DenseMatrix b = random_matrix(25, 18, 3);
    const rsvd::SvdApprox f1 = rsvd::rsvd(b, rsvd::SketchConfig{5, 3, 7, rsvd::RangeMode::basic, 11});
    const rsvd::SvdApprox f2 = rsvd::rsvd(b, rsvd::SketchConfig{5, 3, 0, rsvd::RangeMode::power, 11});
    REQUIRE(max_abs_diff(f1.U, f2.U) == 0.0);
    REQUIRE(max_abs_diff(f1.V, f2.V) == 0.0);
    REQUIRE_THROWS_AS(rsvd::truncate(f1, 9), rsvd::DimensionError);
  }
  // test_rangefinder.cpp:38-46
  {
    const DenseMatrix a = DenseMatrix::Identity(6, 4);
    Rng rng(1);
    REQUIRE_THROWS_AS(rsvd::fixed_rank_range(a, 4, 1, rng), rsvd::DimensionError);
    REQUIRE_THROWS_AS(rsvd::power_range(a, 0, 2, 1, rng), rsvd::ParameterError);
    REQUIRE_THROWS_AS(rsvd::power_range(a, 2, 1, -1, rng), rsvd::ParameterError);
  }
  // test_singlepass.cpp:37-44, 96-103
  {
    const DenseMatrix g = random_matrix(40, 40, 8);
    const DenseMatrix s = DenseMatrix(g * DenseMatrix::Identity(40, 40));
    DenseMatrix sym(40, 40);
    for (int j = 0; j < 40; ++j)
      for (int i = 0; i < 40; ++i) sym(i, j) = 0.5 * (s(i, j) + s(j, i));
    rsvd::CountingOperator op(sym);
    Rng rng(2);
    rsvd::spevd_hermitian(op, 5, 3, rng);
    REQUIRE(op.apply_count() == 1);
    REQUIRE(op.adjoint_count() == 0);
    const DenseMatrix a = random_matrix(30, 20, 9);
    rsvd::CountingOperator op2(a);
    Rng rng2(3);
    rsvd::spsvd_general(op2, 4, 3, rng2);
    REQUIRE(op2.apply_count() == 1);
    REQUIRE(op2.adjoint_count() == 1);
    REQUIRE_THROWS_AS(rsvd::spevd_hermitian(random_matrix(6, 6, 2), 2, 1, rng),
                      rsvd::NumericError);
  }
  // diagnostics: spectral_norm (core.hpp:188-221), computed_range_error
  // (bounds.hpp:107-120), canonical_sines / subspace_quality (angles.hpp:42-78)
  {
    DenseMatrix d(600, 600);
    for (int i = 0; i < 600; ++i) d(i, i) = (i == 7) ? 3.0 : 1.0 / (1.0 + i);
    REQUIRE(std::abs(rsvd::spectral_norm(d) - 3.0) <= 1e-9 * 3.0);  // power route
    const DenseMatrix small = random_matrix(40, 30, 4);
    const auto sv = rsvd::singular_values(small);
    REQUIRE(std::abs(rsvd::spectral_norm(small) - sv(0)) <= 1e-14 * sv(0));  // dense route
    const DenseMatrix a = random_matrix(60, 40, 5);
    Rng rng(6);
    const DenseMatrix q = rsvd::fixed_rank_range(a, 10, 5, rng);
    const double err = rsvd::computed_range_error(a, q);
    REQUIRE(err >= sv(0) * 0.0 && err <= rsvd::spectral_norm(a));
    REQUIRE(err >= rsvd::singular_values(a)(15) * (1 - 1e-10));  // Eckart-Young floor
    REQUIRE_THROWS_AS(rsvd::computed_range_error(random_matrix(50, 40, 1), q),
                      rsvd::DimensionError);
    const auto same = rsvd::canonical_sines(q, q);
    REQUIRE(same.rows() == 15);
    for (int i = 0; i < 15; ++i) REQUIRE(std::abs(same(i)) < 1e-13);
    const rsvd::SvdApprox f = rsvd::rsvd(a, rsvd::SketchConfig{5, 5, 2, rsvd::RangeMode::power, 1});
    const rsvd::AngleReport rep = rsvd::subspace_quality(a, 5, f);
    REQUIRE(rep.k == 5 && rep.sin_theta.rows() == 5 && rep.sin_nu.rows() == 5);
    for (int i = 0; i + 1 < 5; ++i) REQUIRE(rep.sin_theta(i) <= rep.sin_theta(i + 1));
    REQUIRE_THROWS_AS(rsvd::subspace_quality(a, 0, f), rsvd::ParameterError);
    REQUIRE_THROWS_AS(rsvd::canonical_sines(a, q), rsvd::NumericError);
  }
  std::printf(g_fail ? "drop-in: %d failures\n" : "drop-in: all passed\n", g_fail);
  return g_fail ? 1 : 0;
}
