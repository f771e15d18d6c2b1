// MT19937-64 jump polynomials (mtjump.cpp).
#pragma once
#include <cstdint>

namespace rsvdb {
namespace mtjump {
// Polynomials x^(s L - 313) mod phi for s = 1..count, count x words() words
// each (bit k = coefficient of x^k).  Pointer valid until the next call.
const uint64_t* jump_polys(uint64_t L, int count);
int degree();
int words();
}  // namespace mtjump
}  // namespace rsvdb
