// MT19937-64 jump-ahead polynomials (host side, seed independent).
//
// The MT19937-64 state transition T acts on a 19937-dimensional GF(2) space
// (upper 33 bits of x[t] and words x[t+1..t+311]).  With phi the characteristic
// polynomial of T and  x^J mod phi = sum_k c_k x^k,  every output word satisfies
//     x[t + 1 + J] = XOR_{k : c_k = 1} x[t + 1 + k]          (t >= 0)
// so the 312-word window that seeds the generator J words ahead is an XOR of
// shifted windows of the first 19937 + 312 words (rng.cu, mt_jump_kernel).
// phi is obtained once per process by Berlekamp-Massey on one output bit of a
// generated sequence (its minimal polynomial has full degree 19937), and the
// jump polynomials by GF(2) polynomial arithmetic (carry-less multiply).
//
// This is the published jump-ahead method for F2-linear generators (Haramoto
// et al., "Efficient jump ahead for F2-linear random number generators").
#include <immintrin.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "mtjump.h"

namespace rsvdb {
namespace mtjump {
namespace {

constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 64) / 64;  // 312 words hold degrees 0..19967
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;

using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

inline uint64_t twist(uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}

// Raw (untempered) word sequence of mt19937_64(seed): x[0..312) = seeded state.
std::vector<uint64_t> sequence(uint64_t seed, size_t n) {
  std::vector<uint64_t> x(n + 312);
  x[0] = seed;
  for (int i = 1; i < 312; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
  for (size_t t = 312; t < x.size(); ++t) x[t] = x[t - 156] ^ twist(x[t - 312], x[t - 311]);
  return x;
}

// Berlekamp-Massey over GF(2); returns the connection polynomial C (C[0] = 1)
// of the bit sequence s, as a vector of bits.
std::vector<uint8_t> berlekamp_massey(const std::vector<uint8_t>& s) {
  const size_t n = s.size();
  std::vector<uint8_t> C(n + 1, 0), B(n + 1, 0), T;
  C[0] = B[0] = 1;
  size_t L = 0, m = 1;
  for (size_t i = 0; i < n; ++i) {
    uint8_t d = s[i];
    for (size_t j = 1; j <= L; ++j) d ^= C[j] & s[i - j];
    if (d == 0) {
      ++m;
    } else if (2 * L <= i) {
      T = C;
      for (size_t j = 0; j + m <= n; ++j) C[j + m] ^= B[j];
      L = i + 1 - L;
      B = T;
      m = 1;
    } else {
      for (size_t j = 0; j + m <= n; ++j) C[j + m] ^= B[j];
      ++m;
    }
  }
  C.resize(L + 1);
  return C;
}

struct Ctx {
  Poly phi;                 // degree kDeg, monic
  std::vector<Poly> phis;   // phi << s for s = 0..63 (word-aligned reduction)
};

Ctx build_ctx() {
  // bit 0 of x[t + 1], t >= 0 (any fixed seed)
  const size_t n = 2 * kDeg + 64;
  std::vector<uint64_t> x = sequence(5489ULL, n + 2);
  std::vector<uint8_t> s(n);
  for (size_t t = 0; t < n; ++t) s[t] = uint8_t(x[t + 1] & 1ULL);
  std::vector<uint8_t> C = berlekamp_massey(s);
  if (C.size() != size_t(kDeg) + 1) throw std::runtime_error("mtjump: unexpected linear complexity");
  // characteristic polynomial = reciprocal of the connection polynomial
  Ctx c;
  c.phi.assign(kWords + 1, 0);
  for (int i = 0; i <= kDeg; ++i)
    if (C[size_t(kDeg - i)]) c.phi[size_t(i) / 64] |= 1ULL << (i % 64);
  c.phis.resize(64);
  for (int sft = 0; sft < 64; ++sft) {
    Poly p(kWords + 2, 0);
    for (int w = 0; w <= kWords; ++w) {
      p[size_t(w)] ^= c.phi[size_t(w)] << sft;
      if (sft && w + 1 < int(p.size())) p[size_t(w) + 1] ^= c.phi[size_t(w)] >> (64 - sft);
    }
    c.phis[size_t(sft)] = std::move(p);
  }
  return c;
}

const Ctx& ctx() {
  static Ctx c;
  static std::once_flag once;
  std::call_once(once, [] { c = build_ctx(); });
  return c;
}

inline bool bit(const Poly& p, int i) { return (p[size_t(i) / 64] >> (i % 64)) & 1ULL; }

// r (up to 2*kWords words) mod phi, in place; result in the low kWords words.
void reduce(Poly& r) {
  const Ctx& c = ctx();
  for (int i = int(r.size()) * 64 - 1; i >= kDeg; --i) {
    if (!bit(r, i)) continue;
    const int sh = i - kDeg;  // XOR phi * x^sh
    const int w0 = sh / 64, b = sh % 64;
    const Poly& ps = c.phis[size_t(b)];
    for (size_t w = 0; w < ps.size() && w0 + w < r.size(); ++w) r[w0 + w] ^= ps[w];
  }
  r.resize(kWords);
}

inline void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  const __m128i x = _mm_set_epi64x(0, static_cast<long long>(a));
  const __m128i y = _mm_set_epi64x(0, static_cast<long long>(b));
  const __m128i z = _mm_clmulepi64_si128(x, y, 0x00);
  lo = static_cast<uint64_t>(_mm_cvtsi128_si64(z));
  hi = static_cast<uint64_t>(_mm_extract_epi64(z, 1));
}

Poly mulmod(const Poly& a, const Poly& b) {
  Poly r(2 * kWords + 1, 0);
  for (int i = 0; i < kWords; ++i) {
    if (!a[size_t(i)]) continue;
    for (int j = 0; j < kWords; ++j) {
      if (!b[size_t(j)]) continue;
      uint64_t lo, hi;
      clmul64(a[size_t(i)], b[size_t(j)], lo, hi);
      r[size_t(i + j)] ^= lo;
      r[size_t(i + j) + 1] ^= hi;
    }
  }
  reduce(r);
  return r;
}

Poly x_pow(uint64_t e) {  // x^e mod phi, left-to-right square-and-multiply
  Poly r(kWords, 0);
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    r = mulmod(r, r);
    if ((e >> b) & 1ULL) {  // multiply by x
      Poly t(kWords + 1, 0);
      for (int w = 0; w < kWords; ++w) {
        t[size_t(w)] ^= r[size_t(w)] << 1;
        t[size_t(w) + 1] ^= r[size_t(w)] >> 63;
      }
      reduce(t);
      r = t;
    }
  }
  return r;
}

struct Table {
  uint64_t L = 0;
  Poly step;                  // x^L
  std::vector<Poly> polys;    // polys[s-1] = x^(s L - 313), s >= 1
};

}  // namespace

const uint64_t* jump_polys(uint64_t L, int count) {
  static std::mutex mu;
  static std::vector<Table> tabs;  // one table per segment length
  std::lock_guard<std::mutex> lk(mu);
  Table* tp = nullptr;
  for (auto& t : tabs)
    if (t.L == L) tp = &t;
  if (!tp) {
    tabs.push_back(Table{});
    tp = &tabs.back();
    tp->L = L;
    tp->step = x_pow(L);
  }
  Table& tab = *tp;
  while (int(tab.polys.size()) < count) {
    if (tab.polys.empty())
      tab.polys.push_back(x_pow(L - 313));
    else
      tab.polys.push_back(mulmod(tab.polys.back(), tab.step));
  }
  // contiguous copy (count x kWords words), stable until the next call
  static std::vector<uint64_t> flat;
  flat.assign(size_t(count) * kWords, 0);
  for (int s = 0; s < count; ++s)
    std::memcpy(flat.data() + size_t(s) * kWords, tab.polys[size_t(s)].data(), kWords * 8);
  return flat.data();
}

int degree() { return kDeg; }
int words() { return kWords; }

}  // namespace mtjump
}  // namespace rsvdb
