// Register-level primitives of the fused detector: bit-sliced compare,
// bit-plane transposition, segment test, FMA-pipe shifts, packed SAD.
#pragma once

#include <cstdint>

#include "fast_math.cuh"

namespace flkb {
namespace fused {

// ------------------------------------------------------------ primitives

__device__ __forceinline__ uint32_t lop3_maj_na(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;  // (~a & b) | (~a & c) | (b & c): borrow of a - b - c
  asm("lop3.b32 %0, %1, %2, %3, 0x8E;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3_maj(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// Shifts on the FMA pipe (IMAD), leaving the ALU pipe -- which issues at half
// rate and carries every LOP3 -- to the bit-sliced logic:
// x >> k = mulhi(x, 2^(32-k)); x << k = mullo(x, 2^k), with 2^k read from the
// constant bank so ptxas cannot strength-reduce it back into SHF.
template <int K>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << (32 - K)));
  return d;
}
__device__ __forceinline__ uint32_t shl_fma(uint32_t x, uint32_t pow2k) {
  uint32_t d;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(pow2k));
  return d;
}
// Ring-plane shift by a (compile-time after unrolling) dx in [-3, 3]: bit b
// of the result holds bit b + dx of x.
__device__ __forceinline__ uint32_t shift_fma(uint32_t x, int dx, const uint32_t (&pow2)[32]) {
  switch (dx) {
    case 1: return shr_fma<1>(x);
    case 2: return shr_fma<2>(x);
    case 3: return shr_fma<3>(x);
    case -1: return shl_fma(x, pow2[1]);
    case -2: return shl_fma(x, pow2[2]);
    case -3: return shl_fma(x, pow2[3]);
    default: return x;
  }
}
__device__ __forceinline__ uint32_t and3(uint32_t a, uint32_t b, uint32_t c) { return a & b & c; }
__device__ __forceinline__ uint32_t or3(uint32_t a, uint32_t b, uint32_t c) { return a | b | c; }

// Bit-sliced unsigned a < b over 8 planes (plane 0 = LSB): borrow out of a - b.
__device__ __forceinline__ uint32_t sliced_less(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
  uint32_t br = ~a[0] & b[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) br = lop3_maj_na(a[k], b[k], br);
  return br;
}

// 32 pixels (8 words, pixel 4m+i in byte i of word m) -> 8 bit planes.
__device__ __forceinline__ void transpose32x8(const uint32_t (&w)[8], uint32_t (&p)[8],
                                              const uint32_t (&pow2)[32]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    uint32_t l = w[2 * t], h = w[2 * t + 1], x;
    x = (l ^ shr_fma<7>(l)) & 0x00AA00AAu;
    l = l ^ x ^ shl_fma(x, pow2[7]);
    x = (h ^ shr_fma<7>(h)) & 0x00AA00AAu;
    h = h ^ x ^ shl_fma(x, pow2[7]);
    x = (l ^ shr_fma<14>(l)) & 0x0000CCCCu;
    l = l ^ x ^ shl_fma(x, pow2[14]);
    x = (h ^ shr_fma<14>(h)) & 0x0000CCCCu;
    h = h ^ x ^ shl_fma(x, pow2[14]);
    x = (l ^ shl_fma(h, pow2[4])) & 0xF0F0F0F0u;
    l ^= x;
    h ^= shr_fma<4>(x);
    lo[t] = l;
    hi[t] = h;
  }
  // 4x4 byte transposes: plane k byte t = block t byte k
  uint32_t a = __byte_perm(lo[0], lo[1], 0x5140), b = __byte_perm(lo[0], lo[1], 0x7362);
  uint32_t c = __byte_perm(lo[2], lo[3], 0x5140), d = __byte_perm(lo[2], lo[3], 0x7362);
  p[0] = __byte_perm(a, c, 0x5410);
  p[1] = __byte_perm(a, c, 0x7632);
  p[2] = __byte_perm(b, d, 0x5410);
  p[3] = __byte_perm(b, d, 0x7632);
  a = __byte_perm(hi[0], hi[1], 0x5140);
  b = __byte_perm(hi[0], hi[1], 0x7362);
  c = __byte_perm(hi[2], hi[3], 0x5140);
  d = __byte_perm(hi[2], hi[3], 0x7362);
  p[4] = __byte_perm(a, c, 0x5410);
  p[5] = __byte_perm(a, c, 0x7632);
  p[6] = __byte_perm(b, d, 0x5410);
  p[7] = __byte_perm(b, d, 0x7632);
}

// Bit-sliced segment test: some cyclic run of >= N set positions among the
// 16 position words (bit lanes = pixels).
template <int N>
__device__ __forceinline__ uint32_t sliced_arc(const uint32_t (&m)[16]) {
  uint32_t w3[16], w9[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w3[i] = and3(m[i], m[(i + 1) & 15], m[(i + 2) & 15]);
#pragma unroll
  for (int i = 0; i < 16; ++i) w9[i] = and3(w3[i], w3[(i + 3) & 15], w3[(i + 6) & 15]);
  if (N > 9) {
#pragma unroll
    for (int i = 0; i < 16; ++i) w3[i] = w9[i] & w9[(i + N - 9) & 15];
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) w3[i] = w9[i];
  }
  uint32_t a = or3(w3[0], w3[1], w3[2]), b = or3(w3[3], w3[4], w3[5]);
  uint32_t c = or3(w3[6], w3[7], w3[8]), d = or3(w3[9], w3[10], w3[11]);
  uint32_t e = or3(w3[12], w3[13], w3[14]);
  return or3(or3(a, b, c), or3(d, e, w3[15]), 0u);
}

__device__ __forceinline__ uint32_t vabsdiff4_acc(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

// SAD-B of one corner from its 16 ring bytes packed 4 per word:
// sum max(|d|-e,0) = (sum | |d| - e | + sum |d| - 16 e) / 2.
__device__ __forceinline__ int sad_b_packed(const uint32_t (&r)[4], uint32_t c, uint32_t eps) {
  const uint32_t c4 = c * 0x01010101u, e4 = eps * 0x01010101u;
  uint32_t acc1 = 0, acc2 = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t d = __vabsdiffu4(r[k], c4);
    acc1 = vabsdiff4_acc(d, e4, acc1);
    acc2 = vabsdiff4_acc(r[k], c4, acc2);
  }
  return static_cast<int>((acc1 + acc2 - 16u * eps) >> 1);
}

}  // namespace fused
}  // namespace flkb
