// Per-pixel FAST arithmetic shared by the kernels.
//
// The reference decides the segment test with an 8 KB bit table
// (fast.cpp:34-65, 221-247) and scores with loops (fast.cpp:123-203). On
// sm_100a the same answers come out of register-only bit algebra:
//   arc test   doubled 32-bit mask, run-length doubling: AND of shifted
//              copies (run >= 2, 4, 8, then N); identical to
//              has_cyclic_run for every mask and N in [9,16]
//   SAD-B      sum of max(|I_i - c| - eps, 0)                (fast.cpp:156-163)
//   SAD-A      the same terms over the union of full N-windows inside the
//              qualifying mask -- equals best_arc_sum since at most one run
//              of >= 9 fits in 16 positions                  (fast.cpp:123-154)
//   MT         max over polarity and window start of the window minimum of
//              the signed difference, minus 1 -- equals the binary search of
//              max_threshold_score, because the segment test at threshold t
//              passes iff that maximin exceeds t             (fast.cpp:168-181)
// The 16-bit SIMD min/max (VIMNMX.U16x2) evaluates both polarities at once.
#pragma once

#include <cstdint>

#include "../../include/fastlk.h"

namespace flkb {

// kBresenhamCircle (fast.cpp:13-16), clockwise from (0,-3), y down.
__host__ __device__ __forceinline__ constexpr int ring_dx(int i) {
  return i == 0 ? 0 : i == 1 ? 1 : i == 2 ? 2 : i == 3 ? 3 : i == 4 ? 3 : i == 5 ? 3 : i == 6 ? 2
       : i == 7 ? 1 : i == 8 ? 0 : i == 9 ? -1 : i == 10 ? -2 : i == 11 ? -3 : i == 12 ? -3
       : i == 13 ? -3 : i == 14 ? -2 : -1;
}
__host__ __device__ __forceinline__ constexpr int ring_dy(int i) { return ring_dx((i + 12) & 15); }

enum : int { kSadB = 0, kSadA = 1, kMt = 2 };

// Bit i of the result (i < 16) is set iff the cyclic 16-bit mask has bits
// i..i+N-1 all set.
template <int N>
__device__ __forceinline__ uint32_t run_starts(uint32_t m16) {
  uint32_t a = m16 | (m16 << 16);
  a &= a >> 1;
  a &= a >> 2;
  a &= a >> 4;
  a &= a >> (N - 8);
  return a & 0xFFFFu;
}

// Positions covered by the N-windows starting at the bits of `starts`.
template <int N>
__device__ __forceinline__ uint32_t cover_of(uint32_t starts) {
  uint32_t c = starts | (starts << 1);
  c |= c << 2;
  c |= c << 4;
  c |= c << (N - 8);
  return (c | (c >> 16)) & 0xFFFFu;
}

template <int N, int KIND>
__device__ __forceinline__ int fast_score(int c, const int (&ring)[16], int eps) {
  const int lo = c - eps, hi = c + eps;
  uint32_t dark = 0, bright = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    dark |= static_cast<uint32_t>(ring[i] < lo) << i;
    bright |= static_cast<uint32_t>(ring[i] > hi) << i;
  }
  const uint32_t sd = run_starts<N>(dark), sb = run_starts<N>(bright);
  if ((sd | sb) == 0) return 0;
  if (KIND == kSadB) {
    int sum = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) sum += max(abs(ring[i] - c) - eps, 0);
    return sum;
  } else if (KIND == kSadA) {
    const uint32_t cov = cover_of<N>(sd | sb);
    int sum = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) sum += ((cov >> i) & 1u) ? max(abs(ring[i] - c) - eps, 0) : 0;
    return sum;
  } else {
    // lanes: low = c - I + 256 (dark), high = I - c + 256 (bright)
    uint32_t v[16], m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      v[i] = static_cast<uint32_t>(c - ring[i] + 256) | (static_cast<uint32_t>(ring[i] - c + 256) << 16);
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = __vminu2(v[i], v[(i + 1) & 15]);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __vminu2(m[i], m[(i + 2) & 15]);
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = __vminu2(v[i], v[(i + 4) & 15]);
    uint32_t best = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) best = __vmaxu2(best, __vminu2(m[i], m[(i + N - 8) & 15]));
    const int M = max(static_cast<int>(best & 0xFFFFu), static_cast<int>(best >> 16)) - 256;
    return M - 1;
  }
}

// 2x2 round-half-up means (image.cpp:50-62) of two rows of 8 pixels each
// (a0 a1 = row 0, b0 b1 = row 1, pixel 4m+i in byte i of word m) -> 4 output
// bytes. Byte pairs are spread into 16-bit lanes with PRMT, summed with
// IADD3 (at most 4*255+2, no carry between lanes), and bytes 0 and 2 of the
// lanes shifted right by 2 are the means.
__device__ __forceinline__ uint32_t down4(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  const uint32_t s0 = __byte_perm(a0, 0, 0x7250) + __byte_perm(a0, 0, 0x7351) +
                      __byte_perm(b0, 0, 0x7250) + __byte_perm(b0, 0, 0x7351) + 0x00020002u;
  const uint32_t s1 = __byte_perm(a1, 0, 0x7250) + __byte_perm(a1, 0, 0x7351) +
                      __byte_perm(b1, 0, 0x7250) + __byte_perm(b1, 0, 0x7351) + 0x00020002u;
  return __byte_perm(s0 >> 2, s1 >> 2, 0x6420);
}

// cell_candidate_wins (nms.cpp:41-46) as one unsigned compare: higher score,
// then lower level, then smaller y0, then smaller x0.
__device__ __forceinline__ unsigned long long pack_key(int score, int level, int x0, int y0) {
  constexpr unsigned long long kMask = (1ull << 18) - 1ull;
  return (static_cast<unsigned long long>(score) << 40) |
         (static_cast<unsigned long long>(15 - level) << 36) |
         ((kMask - static_cast<unsigned long long>(y0)) << 18) |
         (kMask - static_cast<unsigned long long>(x0));
}

__device__ __forceinline__ flk_feature unpack_key(unsigned long long key, int cx, int cy) {
  constexpr unsigned long long kMask = (1ull << 18) - 1ull;
  flk_feature f;
  f.x = static_cast<int>(kMask - (key & kMask));
  f.y = static_cast<int>(kMask - ((key >> 18) & kMask));
  f.level = 15 - static_cast<int>((key >> 36) & 15ull);
  f.score = static_cast<float>(static_cast<int>(key >> 40));
  f.cell_x = cx;
  f.cell_y = cy;
  return f;
}

// ------------------------------------------------------ synthetic frames

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t synth_hash(uint64_t f, uint64_t i, uint64_t salt) {
  return splitmix64(0x200313493ull ^ (f << 32) ^ i ^ (salt << 60));
}
__host__ __device__ __forceinline__ uint8_t synth_pixel(int kind, uint64_t f, int x, int y, int w) {
  if (kind == 0) return static_cast<uint8_t>(synth_hash(f, static_cast<uint64_t>(y) * w + x, 0));
  const uint64_t gw = static_cast<uint64_t>(w / 8 + 2);
  const uint64_t gx = static_cast<uint64_t>(x >> 3), gy = static_cast<uint64_t>(y >> 3);
  const int64_t v00 = 30 + static_cast<int64_t>(synth_hash(f, gy * gw + gx, 1) % 160);
  const int64_t v10 = 30 + static_cast<int64_t>(synth_hash(f, gy * gw + gx + 1, 1) % 160);
  const int64_t v01 = 30 + static_cast<int64_t>(synth_hash(f, (gy + 1) * gw + gx, 1) % 160);
  const int64_t v11 = 30 + static_cast<int64_t>(synth_hash(f, (gy + 1) * gw + gx + 1, 1) % 160);
  const int64_t wx = (x & 7) * 32, wy = (y & 7) * 32;
  const int64_t top = v00 * (256 - wx) + v10 * wx;
  const int64_t bot = v01 * (256 - wx) + v11 * wx;
  int64_t val = (top * (256 - wy) + bot * wy + 32768) >> 16;
  val += static_cast<int64_t>(synth_hash(f, static_cast<uint64_t>(y) * w + x, 2) % 7) - 3;
  return static_cast<uint8_t>(val < 0 ? 0 : (val > 255 ? 255 : val));
}

}  // namespace flkb
