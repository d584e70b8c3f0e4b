// Native config generator: the reference's preferential-attachment graph
// (testkit.py:175-198) reproduced draw-for-draw in C++ so configs C2/C4
// (1e6 / 2e6 nodes) are built in well under a second instead of a Python
// loop.  The draw stream is numpy's PCG64 (XSL-RR 128/64, state advanced
// before output) consumed as numpy's Generator.integers(0, L) does for a
// scalar bound L <= 2^32: one 32-bit word per attempt (low half of a 64-bit
// output first, the high half kept for the next call), Lemire's multiply-shift
// with rejection below (2^32 - L) mod L.  Pinned against numpy by
// tests/test_host.py (SHA-256 of the full C2/C4 graphs in tests/golden).
#include <stdint.h>

#include <vector>

#include "../../include/kpm.h"

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t u32;

  uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }

  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }

  // Generator.integers(0, bound) for 2 <= bound <= 2^32 (scalar call)
  uint64_t bounded(uint64_t bound) {
    const uint32_t excl = (uint32_t)bound;  // bound == 2^32 is not used here
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thresh = (uint32_t)(-excl) % excl;
      while (left < thresh) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
};

}  // namespace

extern "C" int kpm_gen_preferential_attachment(int64_t n, int64_t m, const uint64_t *pcg,
                                               int64_t *u, int64_t *v) {
  if (m < 1 || m >= n || !pcg || !u || !v) return KPM_EINVAL;
  Pcg64 g;
  g.state = ((unsigned __int128)pcg[0] << 64) | pcg[1];
  g.inc = ((unsigned __int128)pcg[2] << 64) | pcg[3];
  g.has32 = (int)pcg[4];
  g.u32 = (uint32_t)pcg[5];
  const int64_t n_edges = m * (m + 1) / 2 + (n - m - 1) * m;
  if (2 * n_edges > (int64_t(1) << 32)) return KPM_EINVAL;  // 32-bit draw path only
  std::vector<int64_t> ends(2 * n_edges);
  int64_t e = 0;
  for (int64_t a = 0; a <= m; ++a)
    for (int64_t b = a + 1; b <= m; ++b) {
      u[e] = a;
      v[e] = b;
      ends[2 * e] = a;
      ends[2 * e + 1] = b;
      ++e;
    }
  std::vector<int64_t> picked;
  picked.reserve(m);
  for (int64_t node = m + 1; node < n; ++node) {
    const uint64_t len = (uint64_t)(2 * e);
    picked.clear();
    while ((int64_t)picked.size() < m) {
      int64_t t = ends[g.bounded(len)];
      bool seen = false;
      for (int64_t x : picked) seen |= (x == t);
      if (!seen) picked.push_back(t);
    }
    // sorted(targets): m is small, insertion sort
    for (size_t i = 1; i < picked.size(); ++i)
      for (size_t j = i; j > 0 && picked[j - 1] > picked[j]; --j) {
        int64_t t = picked[j];
        picked[j] = picked[j - 1];
        picked[j - 1] = t;
      }
    for (int64_t t : picked) {
      u[e] = t;
      v[e] = node;
      ends[2 * e] = t;
      ends[2 * e + 1] = node;
      ++e;
    }
  }
  return KPM_OK;
}
