// Measures how far from a rounding midpoint log(r2) must lie for glibc's log
// to differ from the correctly rounded value, over the reference's own polar
// inputs (mt19937_64 + generate_canonical + 2u-1, libstdc++ random.tcc).
//
// For every accepted r2 it evaluates the double-double log (csrc/ddlog.cuh,
// ~2^-75 relative), the distance d (in ulps of the rounded result) between the
// exact value and the nearest rounding midpoint, and glibc's std::log.  It
// prints the mismatch count, the largest d among mismatches, and the number
// of inputs a window W would flag, for the windows the engine may use.
//
//   g++ -O2 -std=c++17 -mfma -pthread -I paper_2402_17794_b200/csrc \
//       tools/logwindow.cpp -o /tmp/logwindow
//   /tmp/logwindow <pairs_per_thread> <threads> [seed0]
// Run once per glibc ifunc variant (default, and with
// GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2_Usable,-FMA_Usable,-AVX2,-FMA).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "ddlog.cuh"

using namespace rsvdb::ddlog;

namespace {
struct Stat {
  long long accepted = 0, mismatch = 0, pow2 = 0;
  double max_d_mismatch = 0.0;  // largest midpoint distance (ulps) of a mismatch
  long long flagged[4] = {0, 0, 0, 0};
  // per binade of log(r2) (exponent e of |log r2| = f*2^e, e in [-60, 10)):
  double max_d_bin[70] = {0};
  long long mism_bin[70] = {0}, acc_bin[70] = {0};
  long long model_flagged = 0, model_miss = 0;  // engine window w(e) (ddlog.cuh)
  double model_margin = 1e300;  // min over mismatches of w(e) / d
};
const double kWin[4] = {1.0 / 256, 1.0 / 128, 1.0 / 64, 1.0 / 32};

// The engine's flag test, restated (rng.cu log_near_midpoint).
double mid_distance(double x, const Entry* tab, double* v, bool* p2) {
  const dd s = log_dd(x, tab);
  *v = s.hi + s.lo;
  return midpoint_distance(s, *v, p2);
}
}  // namespace

int main(int argc, char** argv) {
  const long long per = argc > 1 ? atoll(argv[1]) : 1000000;
  const int nt = argc > 2 ? atoi(argv[2]) : 8;
  const unsigned long long seed0 = argc > 3 ? strtoull(argv[3], nullptr, 10) : 1;
  static Entry tab[kTableSize];
  build_table(tab);
  std::vector<Stat> st(nt);
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      std::mt19937_64 g(seed0 + t);
      Stat& s = st[t];
      for (long long i = 0; i < per; ++i) {
        const double x = 2.0 * std::generate_canonical<double, 53>(g) - 1.0;
        const double y = 2.0 * std::generate_canonical<double, 53>(g) - 1.0;
        const double r2 = x * x + y * y;
        if (r2 > 1.0 || r2 == 0.0) continue;
        ++s.accepted;
        double v;
        bool p2;
        const double d = mid_distance(r2, tab, &v, &p2);
        if (p2) ++s.pow2;
        int eb = 0;
        frexp(v, &eb);
        const int bi = eb < -60 ? 0 : (eb >= 10 ? 69 : eb + 60);
        ++s.acc_bin[bi];
        for (int w = 0; w < 4; ++w)
          if (p2 || d < kWin[w]) ++s.flagged[w];
        const dd sd = log_dd(r2, tab);
        const bool fl = log_near_midpoint(sd, v);
        if (fl) ++s.model_flagged;
        if (std::log(r2) != v) {
          if (!fl) {
            ++s.model_miss;
            printf("MODEL MISS: r2=%a glibc=%a cr=%a d=%.6f\n", r2, std::log(r2), v, d);
          } else if (!p2) {
            const double w = ldexp(0.04, -std::abs(eb + 3));
            if (w / d < s.model_margin) s.model_margin = w / d;
          }
          ++s.mismatch;
          ++s.mism_bin[bi];
          if (d > s.max_d_bin[bi]) s.max_d_bin[bi] = d;
          if (d > s.max_d_mismatch) s.max_d_mismatch = d;
        }
      }
    });
  for (auto& x : th) x.join();
  Stat tot;
  for (auto& s : st) {
    tot.accepted += s.accepted;
    tot.mismatch += s.mismatch;
    tot.pow2 += s.pow2;
    tot.model_flagged += s.model_flagged;
    tot.model_miss += s.model_miss;
    tot.model_margin = std::fmin(tot.model_margin, s.model_margin);
    tot.max_d_mismatch = std::fmax(tot.max_d_mismatch, s.max_d_mismatch);
    for (int w = 0; w < 4; ++w) tot.flagged[w] += s.flagged[w];
    for (int b = 0; b < 70; ++b) {
      tot.acc_bin[b] += s.acc_bin[b];
      tot.mism_bin[b] += s.mism_bin[b];
      tot.max_d_bin[b] = std::fmax(tot.max_d_bin[b], s.max_d_bin[b]);
    }
  }
  for (int b = 0; b < 70; ++b)
    if (tot.acc_bin[b])
      fprintf(stderr, "binade e=%d (|log| in [2^%d,2^%d)): accepted %lld mismatch %lld max_d %.3g\n",
              b - 60, b - 61, b - 60, tot.acc_bin[b], tot.mism_bin[b], tot.max_d_bin[b]);
  printf("{\"attempts\": %lld, \"accepted\": %lld, \"mismatch\": %lld, \"pow2\": %lld, "
         "\"max_mid_distance_of_mismatch_ulp\": %.6g",
         per * nt, tot.accepted, tot.mismatch, tot.pow2, tot.max_d_mismatch);
  for (int w = 0; w < 4; ++w)
    printf(", \"flagged_w%d\": %lld", int(1.0 / kWin[w]), tot.flagged[w]);
  printf(", \"model_window_flagged\": %lld, \"model_window_misses\": %lld, "
         "\"model_window_min_margin\": %.3f}\n",
         tot.model_flagged, tot.model_miss, tot.model_margin);
  return 0;
}
