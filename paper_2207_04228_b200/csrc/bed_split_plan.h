// bed_split_plan.h -- workspace layout and chunking of the medium path
// (9 <= n <= 64); host-only arithmetic shared by the launcher
// (bed_split_launch.cuh) and the C ABI's workspace query (bed_capi.cu).
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <algorithm>

namespace bed {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Tier order (NMAX) of the medium path for n in [9, 64].
inline int split_nmax(int n) { return n <= 16 ? 16 : (n <= 24 ? 24 : (n <= 32 ? 32 : 64)); }
// Workspace of one chunk of Bc matrices (Bc a multiple of 32), carved from one
// caller-provided block: P (the initial V), the band, the validation status
// and, with vectors, the rotation record Q writes and F reads, which holds
// every sweep the double-step budget allows (2 * max_steps + 1).
struct SplitPlan {
  int64_t Bc = 0;
  size_t bytes = 0, oP = 0, oD = 0, oE = 0, oL = 0, oV = 0, oR = 0, oM = 0, oN = 0, oML = 0;
};

inline SplitPlan split_plan(int64_t Bc, int n, bool vecs, int max_steps) {
  const int nmax = split_nmax(n);
  const bool rec = vecs;
  const size_t smax = 2 * (size_t)max_steps + 1;
  const size_t W = (size_t)Bc / 32, nn = (size_t)n * n;
  SplitPlan p;
  p.Bc = Bc;
  auto take = [&](size_t bytes) {
    size_t o = p.bytes;
    p.bytes += align256(bytes);
    return o;
  };
  p.oP = vecs ? take(4 * (size_t)Bc * nn) : 0;
  p.oD = take(4 * (size_t)Bc * n);
  p.oE = take(4 * (size_t)Bc * n);
  p.oL = rec ? take(4 * (size_t)Bc * n) : 0;
  p.oV = take(4 * (size_t)Bc);
  p.oR = rec ? take(W * smax * (nmax - 1) * 32 * 8) : 0;
  p.oM = rec ? take(W * smax * 4) : 0;
  p.oN = rec ? take(W * 4) : 0;
  p.oML = rec ? take(W * smax * 32) : 0;
  return p;
}

// The largest chunk (multiple of 32, at most the batch rounded up) whose
// workspace fits in `bytes`; 0 if not even 32 matrices fit.
inline int64_t split_chunk(int64_t batch, int n, bool vecs, int max_steps, size_t bytes) {
  const int64_t want = (batch + 31) / 32 * 32;
  if (split_plan(want, n, vecs, max_steps).bytes <= bytes) return want;
  const size_t per32 = split_plan(32, n, vecs, max_steps).bytes;
  int64_t bc = per32 <= bytes ? std::min<int64_t>(want, (int64_t)(bytes / per32) * 32) : 0;
  while (bc > 32 && split_plan(bc, n, vecs, max_steps).bytes > bytes) bc -= 32;
  return split_plan(bc > 0 ? bc : 32, n, vecs, max_steps).bytes <= bytes ? bc : 0;
}

}  // namespace bed
