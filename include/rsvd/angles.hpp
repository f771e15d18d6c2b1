// Drop-in for the reference header of the same name (proj/include/rsvd/angles.hpp (canonical_sines, subspace_quality, AngleReport)),
// executed by the B200 engine.
#pragma once
#include "rsvd_b200.hpp"
