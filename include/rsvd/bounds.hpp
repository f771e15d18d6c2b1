// Drop-in for the reference header of the same name (proj/include/rsvd/bounds.hpp (computed_range_error only: the bound formulas are out of scope)),
// executed by the B200 engine.
#pragma once
#include "rsvd_b200.hpp"
