// Drop-in for the reference header of the same name (proj/include/rsvd/sketch.hpp):
// the hot-path API, executed by the B200 engine.
#pragma once
#include "rsvd_b200.hpp"
