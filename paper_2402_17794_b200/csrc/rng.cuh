// Device Gaussian stream (rng.cu).
#pragma once
#include "common.cuh"
#include "ddlog.cuh"

namespace rsvdb {

// Device-resident copy of the reference Rng state (layout = rsvd_rng_state).
struct DevRng {
  void* d = nullptr;   // DevState on device
  int has_cached = 0;  // host mirror (needed to size the next draw)
};

void rng_init_device(Handle& h);
DevRng rng_upload(Handle& h, const rsvd_rng_state* st);
// Queue the device state for copy-back into *user at the call's final sync.
void rng_download(Handle& h, const DevRng& r, rsvd_rng_state* user);
// n x l normals, column-major into out (rows [row_lo, row_hi) only when
// row_hi >= 0; out then holds row_hi - row_lo rows).  Advances rng.
void gaussian_dev(Handle& h, int64_t n, int64_t l, DevRng& rng, DMat out, int64_t row_lo = 0,
                  int64_t row_hi = -1);
const ddlog::Entry* host_log_table();

}  // namespace rsvdb
