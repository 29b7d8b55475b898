// Fused FAST + score + window-max suppression + cell selection, one CTA per
// (frame, level, band of rows, column tile). sm_100a.
//
//  1. TMA   cp.async.bulk copies the tile's image rows (+3+n halo) of level k
//           from HBM into shared memory, completion on an mbarrier.
//  2. SLICE every 32-byte window (stride 26 px) is transposed into 8 bit
//           planes: bit b of plane k = bit k of pixel x0+b. A word "owns"
//           its middle 26 pixels, so every ring offset (|dx| <= 3) stays
//           inside the word -- no neighbour exchange.
//  3. MASKS bit-sliced FAST: per word, thresholds L = sat(c-eps) and
//           H = sat(c+eps) as 8 planes each, then for each of the 16 ring
//           positions the shifted ring planes are compared with a borrow
//           chain (one LOP3 per bit): dark_i = R_i < L, bright_i = H < R_i,
//           32 pixels per instruction. The segment test is a bit-sliced
//           sliding AND over the 16 position words (runs of 3, then 9, then
//           N) -- 32 pixels' corner decisions per LOP3. Identical to the
//           reference LUT test (fast.cpp:34-65, 221-247).
//  4. SCORE corners are compacted per warp (popc + shuffle scan) and scored
//           one per lane: SAD-B through VABSDIFF4 on packed ring bytes,
//           SAD-A / MT through the register formulations of fast_math.cuh.
//           Scores land in a zero-padded u16 tile in shared memory.
//  5. NMS   each candidate in the band's own rows is tested against its
//           (2n+1)^2 window with spiral_is_local_max's tie rule
//           (nms.cpp:48-79); survivors update a 32-bit per-cell key in
//           shared memory with one ATOMS.MAX (score, -y, -x as offsets inside
//           the CTA; the level is fixed per CTA).
//  6. FLUSH each non-empty cell key becomes the global u64 key (score,
//           -level, -y0, -x0) via one atomicMax -- the cross-level
//           cell_candidate_wins order (nms.cpp:41-46).
#pragma once

#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "fast_math.cuh"

namespace flkb {
namespace fused {

constexpr int kOwn = 26;       // pixels owned by one 32-bit plane word
#ifndef FLKB_THREADS
#define FLKB_THREADS 128
#endif
constexpr int kThreads = FLKB_THREADS;
constexpr int kWarps = kThreads / 32;
#ifndef FLKB_MIN_BLOCKS
#define FLKB_MIN_BLOCKS 6
#endif
constexpr int kMinBlocks = FLKB_MIN_BLOCKS;
#ifndef FLKB_KEYS
#define FLKB_KEYS 0
#endif  // CTAs per SM the register budget targets
constexpr int kMaxLv = 16;
#ifndef FLKB_SCORE_UNROLL
#define FLKB_SCORE_UNROLL 1
#endif
#ifndef FLKB_NMS_UNROLL
#define FLKB_NMS_UNROLL 1
#endif
constexpr int kScoreUnroll = FLKB_SCORE_UNROLL;  // scoring / suppression loop unroll (A/B knobs)
constexpr int kNmsUnroll = FLKB_NMS_UNROLL;
constexpr int kGeoMax = 64;  // CTA geometry entries carried in the launch parameters (1 KB)
// Stage pitch (bytes) and score-tile pitch (u16) of the radius-1 instance:
// column tiles up to 192 px (8 plane words) fit them.
constexpr int kSw1 = 224;
constexpr int kRp1 = 200;
constexpr uint32_t kRpMagic1 = 0xFFFFFFFFu / kRp1 + 1u;  // ceil(2^32 / 200)

// Exact x / d for 0 <= x < 2^31 with one IMAD.HI: q = (umulhi(x, m) + x) >> l,
// l = ceil(log2 d), m = 1 + floor(2^32 (2^l - d) / d).
struct FastDiv {
  uint32_t m = 1;
  int l = 0;
  static FastDiv make(uint32_t d) {
    FastDiv f;
    f.l = 0;
    while ((1ull << f.l) < d) ++f.l;
    f.m = static_cast<uint32_t>(1ull + ((1ull << 32) * ((1ull << f.l) - d)) / d);
    return f;
  }
  __device__ __forceinline__ int operator()(int x) const {
    return static_cast<int>((__umulhi(static_cast<uint32_t>(x), m) + static_cast<uint32_t>(x)) >> l);
  }
};

struct Level {
  // 3-D tiled TMA map of the level (x, y, frame) whose box is one CTA's
  // stage (stage pitch x stage rows): the whole staging is one
  // cp.async.bulk.tensor, rows and columns outside the image zero-filled
  alignas(64) CUtensorMap tmap;
  int tmap_ok;
  const uint8_t* img;  // frame 0, row 0
  size_t fstride;
  int pitch, w, h;
  int tiles_x, tile_w;  // column tiles and NMS columns per tile
  int bands;            // row bands of R rows
  int cta0;             // first blockIdx.x of this level
  int tma;              // rows may be fetched with cp.async.bulk
  int nw;               // plane words per row (max over the level's tiles)
  FastDiv div_nw, div_tiles;
  // grid cell of a level-k pixel: cx = mulhi(x, cmx) + ccx = (x << k) / cell_w,
  // likewise cy (one IMAD.HI each; the host checks every in-image coordinate;
  // ccx, ccy are 0 or 1)
  uint32_t cmx, ccx, cmy, ccy;
  size_t dbg_off;  // diagnostic score dump: level offset (u16 elements) and pitch
  int dbg_pitch;
};

struct Params {
  Level lv[kMaxLv];
  int levels;
  int k_begin, k_end;  // levels detected by this launch (lv[k_begin].cta0 == 0)
  // Pyramid levels 1..pyr_levels (<= 2) written by the level-0 CTAs from their
  // staged rows (needs R % 4 == 0 and 16-px aligned column tiles); 0 = none.
  int pyr_levels;
  uint8_t* pyr_img[3];
  // launched as a programmatic dependent of the pyramid kernel: CTAs of
  // levels >= 1 wait for it (griddepcontrol.wait), level-0 CTAs start at once
  int pdl_wait;  // frame 0, row 0 of levels 1, 2 (index = level)
  int eps, radius, R;
  int cell_w, cell_h, cols, cells;
  FastDiv div_cw, div_ch;
  int sw;         // stage row pitch (bytes)
  int nw_max;     // plane words per row, max over tiles
  int rp;         // score tile pitch (u16)
  uint32_t rp_magic;  // ceil(2^32 / rp): tile row of a tile index e < 2^16 is umulhi(e, rp_magic)
  int key_slots;  // shared cell-key capacity
  int list_cap;   // corner-list capacity (0 = 24 entries per thread)
  uint32_t pow2[32];  // 1 << i, read from the constant bank so shifts can issue as IMAD
  uint32_t emask[8];  // ~0 where bit b of eps is set
  uint32_t neg16eps;  // -16 eps mod 2^32 (SAD-B)
  unsigned long long* keys;
  unsigned long long* stats;
  // diagnostic: when set, every CTA writes the u16 scores of its own rows and
  // columns (the reference's response values, 0 off corners and in the border)
  uint16_t* dbg_map;
  size_t dbg_fstride;
  // stats path only: SM cycles spent by thread 0 of every CTA in the response
  // phases (staging .. scoring) and in the suppression / selection phases,
  // summed, so the host can split the fused launch's time like the
  // reference's crf_us / nms_us (frontend.cpp:42-53)
  unsigned long long* phase_cycles;
  // shared-memory layout and corner-list capacity, filled by the host
  // (finalize()) so the kernel does not recompute them
  int sm_stage, sm_planes, sm_cm, sm_list, sm_scan, sm_skeys, sm_bar, sm_xrow, cap;
  // per-CTA geometry of this launch (host table, geo_n entries; CTAs past it
  // compute theirs): x = k | (cell rows) << 4 | y0 << 16, y = y1 | x_lo << 16,
  // z = x_hi | first cell row << 16, w = first cell column | cell columns << 16
  int geo_n;
  uint4 geo[kGeoMax];
};

struct Smem {
  int stage, planes, cm, list, scan, skeys, bar, xrow, list_entries, total;
};

// Cross-row mask exchange of the mask phase (phase 3): 4 uint4 arrays of
// ring_rows x nw words, ring_rows = kThreads / nw + 3; bounded over nw <= nw_max.
__host__ __device__ inline int xrow_bytes(int nw_max) {
  return 64 * (kThreads + 3 * nw_max);
}

// Corner-list capacity (u16 entries); a band with more corners is scored in
// several rounds.
__host__ __device__ inline int list_capacity(const Params& p) {
  const int worst = (p.R + 2 * p.radius) * p.nw_max * kOwn;
  const int cap = p.list_cap > 0 ? p.list_cap : 24 * kThreads;  // host override (tests force rounds)
  return worst < cap ? (worst + 7) & ~7 : cap;
}

__host__ __device__ inline Smem smem_layout(const Params& p) {
  const int img_rows = p.R + 2 * p.radius + 6;
  const int fast_rows = p.R + 2 * p.radius;
  Smem s;
  int off = 0;
  s.stage = off;
  off += img_rows * p.sw;
  off = (off + 127) & ~127;
  s.planes = off;  // [2 halves][img_rows][nw_max][4 planes]; the score tile aliases it later
  const int pl = img_rows * p.nw_max * 32;
  const int rt = fast_rows * p.rp * 2;
  // the mask phase's cross-row exchange follows the planes; it is dead once
  // the masks exist, so it overlaps the tile's tail and the corner list
  s.xrow = (off + pl + 15) & ~15;
  const int xrow_end = s.xrow + xrow_bytes(p.nw_max);
  off += pl > rt ? pl : rt;
  off = (off + 15) & ~15;
  s.list = off;
  s.list_entries = list_capacity(p);
  if (s.list + 2 * s.list_entries < xrow_end) s.list_entries = ((xrow_end - s.list) / 2 + 7) & ~7;
  off += s.list_entries * 2;
  off = (off + 15) & ~15;
  s.cm = off;
  off += fast_rows * p.nw_max * 4;
  off = (off + 15) & ~15;
  s.scan = off;
  off += (kWarps + 4) * 4;
  off = (off + 15) & ~15;
  s.skeys = off;
  off += p.key_slots * 4;
  off = (off + 15) & ~15;
  s.bar = off;
  off += 32;  // mbarrier + two phase-clock stamps
  s.total = off;
  return s;
}

// Host: stores the layout and list capacity in the parameters the kernel reads.
inline void finalize(Params& p) {
  const Smem s = smem_layout(p);
  p.sm_stage = s.stage;
  p.sm_planes = s.planes;
  p.sm_cm = s.cm;
  p.sm_list = s.list;
  p.sm_scan = s.scan;
  p.sm_skeys = s.skeys;
  p.sm_bar = s.bar;
  p.sm_xrow = s.xrow;
  p.cap = s.list_entries;
}

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
// a * b + c on the FMA pipe (b read from the constant bank so ptxas keeps
// the IMAD rather than strength-reducing it to a shift + add on the ALU pipe)
__device__ __forceinline__ uint32_t mad_fma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
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
// 16 position words (bit lanes = pixels) iff one of the 8 returned words has
// the lane set. With w3[i] = m[i] & m[i+1] & m[i+2], a run starting at i is
// T_i = w3[i] & C_i, C_i = AND m[i+3 .. i+N-1], and the run starting 3 later
// is C_i & w3[i+N]; so T_i | T_{i+3} = C_i & (w3[i] | w3[i+N]). The 16 starts
// pair up along the cycle i -> i+3 (gcd(3, 16) = 1): at N = 9 two LOP3 per
// pair instead of two AND3 and an OR.
template <int N>
__device__ __forceinline__ void sliced_arc_pairs(const uint32_t (&m)[16], uint32_t (&t)[8]) {
  uint32_t w3[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w3[i] = and3(m[i], m[(i + 1) & 15], m[(i + 2) & 15]);
  constexpr int kPair[8] = {0, 6, 12, 2, 8, 14, 4, 10};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = kPair[q];
    uint32_t c = 0xFFFFFFFFu;
    int p = 3;
#pragma unroll
    for (; p + 3 <= N; p += 3) c &= w3[(i + p) & 15];
#pragma unroll
    for (; p < N; ++p) c &= m[(i + p) & 15];
    t[q] = c & (w3[i] | w3[(i + N) & 15]);
  }
}

// Corner lanes of a word: the 16 pair terms of both polarities OR-reduced with
// seven three-input ORs, the last LOP3 also applying the lane mask.
template <int N>
__device__ __forceinline__ uint32_t sliced_corners(const uint32_t (&dk)[16], const uint32_t (&bk)[16],
                                                   uint32_t valid) {
  uint32_t d[8], b[8];
  sliced_arc_pairs<N>(dk, d);
  sliced_arc_pairs<N>(bk, b);
  const uint32_t x = or3(or3(d[0], d[1], d[2]), or3(d[3], d[4], d[5]), or3(d[6], d[7], b[0]));
  const uint32_t y = or3(or3(b[1], b[2], b[3]), or3(b[4], b[5], b[6]), b[7]);
  return (x | y) & valid;
}

__device__ __forceinline__ uint32_t bfind(uint32_t m) {  // index of the highest set bit (FLO)
  uint32_t d;
  asm("bfind.u32 %0, %1;" : "=r"(d) : "r"(m));
  return d;
}
__device__ __forceinline__ uint32_t bit(uint32_t i) {
  uint32_t d;
  asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(d) : "r"(i));  // 1 << i (BMSK, no constant register)
  return d;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t shared_addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(shared_addr) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t vabsdiff4_acc(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

// Twice the SAD-B of one corner from its 16 ring bytes packed 4 per word:
// 2 sum max(|d|-e,0) = sum | |d| - e | + sum |d| - 16 e (the score tile holds
// the doubled scores: the window comparisons are scale-free, and the key's
// score field takes the doubling as one shift less).
// acc0 = -16 e (mod 2^32), a constant-bank operand, starts the first sum.
__device__ __forceinline__ int sad_b_packed(const uint32_t (&r)[4], uint32_t c, uint32_t eps,
                                            uint32_t acc0) {
  const uint32_t c4 = c * 0x01010101u, e4 = eps * 0x01010101u;
  uint32_t acc1 = acc0, acc2 = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t d = __vabsdiffu4(r[k], c4);
    acc1 = vabsdiff4_acc(d, e4, acc1);
    acc2 = vabsdiff4_acc(r[k], c4, acc2);
  }
  return static_cast<int>(acc1 + acc2);
}

// ---------------------------------------------------------------- kernel

// Per-thread walk over a row-major (rows x nw) task grid with stride kThreads,
// without a division per step.
struct TaskIter {
  int row, j, drow, dj, nw;
  __device__ __forceinline__ TaskIter(int t0, int nw_, const FastDiv& div) : nw(nw_) {
    row = div(t0);
    j = t0 - row * nw_;
    drow = div(kThreads);
    dj = kThreads - drow * nw_;
  }
  __device__ __forceinline__ void next() {
    row += drow;
    j += dj;
    if (j >= nw) {
      j -= nw;
      ++row;
    }
  }
};

// STATS: the counting instance (nms_candidates / nms_comparisons, phase
// clocks), used only when flk_frame_stats are requested; the other instance
// carries none of that code.
template <int N, int KIND, int RADIUS, bool STATS>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_detect(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stage / score-tile pitches: compile-time in the radius-1 instance (the host
  // pads the layout to them), so ring and window loads take immediate offsets
  const int SW = RADIUS == 1 ? kSw1 : P.sw;
  const int RP = RADIUS == 1 ? kRp1 : P.rp;
  // SAD-B scores sit doubled in the score tile (sad_b_packed)
  constexpr int kTileShift = KIND == kSadB ? 1 : 0;

  // --- which level, band and column tile: from the host's table of this
  //     launch's CTAs (level, rows, columns, cell range), else computed
  int k, y0, y1, x_lo, x_hi, cr0, nrows, cc0, ccols;
  if (static_cast<int>(blockIdx.x) < P.geo_n) {
    const uint4 g = P.geo[blockIdx.x];
    k = g.x & 15u;
    nrows = (g.x >> 4) & 4095u;
    y0 = g.x >> 16;
    y1 = g.y & 0xFFFFu;
    x_lo = g.y >> 16;
    x_hi = g.z & 0xFFFFu;
    cr0 = g.z >> 16;
    cc0 = g.w & 0xFFFFu;
    ccols = g.w >> 16;
  } else {
    k = P.k_begin;
    while (k + 1 < P.k_end && static_cast<int>(blockIdx.x) >= P.lv[k + 1].cta0) ++k;
    const Level& Lk = P.lv[k];
    const int local = blockIdx.x - Lk.cta0;
    const int band = Lk.div_tiles(local), tile = local - band * Lk.tiles_x;
    y0 = band * P.R;
    y1 = min(y0 + P.R, Lk.h);
    x_lo = tile * Lk.tile_w;
    x_hi = min(x_lo + Lk.tile_w, Lk.w);
    // cell rows touched by the suppressed rows [y0, y1) of level k and the
    // cell columns of its own columns [x_lo, x_hi): the in-CTA keys cover
    // only those cells
    cr0 = P.div_ch(y0 << k);
    nrows = (y1 > y0 ? P.div_ch((y1 - 1) << k) : cr0) - cr0 + 1;
    cc0 = P.div_cw(x_lo << k);
    ccols = (x_hi > x_lo ? P.div_cw((x_hi - 1) << k) : cc0) - cc0 + 1;
  }
  const Level& L = P.lv[k];
  const int f = blockIdx.y;
  const int n = RADIUS > 0 ? RADIUS : P.radius, w = L.w, h = L.h;
  const int fy0 = y0 - n;                                       // tile row 0 <-> image row fy0
  const int iy0 = fy0 - 3;                                      // stage row 0 <-> image row iy0
  const int ya = max(iy0, 0), yb = min(y1 + n + 3, h);          // rows present in the stage
  const int bx0 = (x_lo - n - 3) & ~15;                         // stage column 0 <-> image x bx0
  const int nw = L.nw;                                          // plane words per row
  const int cx_lo = max(x_lo - n, 3), cx_hi = min(x_hi + n, w - 3);  // FAST columns
  const int cy_lo = max(fy0, 3), cy_hi = min(y1 + n, h - 3);         // FAST rows

  uint8_t* stage = smem + P.sm_stage;
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + P.sm_planes);
  uint16_t* tile_s = reinterpret_cast<uint16_t*>(smem + P.sm_planes);
  uint32_t* cm = reinterpret_cast<uint32_t*>(smem + P.sm_cm);
  uint16_t* list = reinterpret_cast<uint16_t*>(smem + P.sm_list);
  int* scan = reinterpret_cast<int*>(smem + P.sm_scan);
  // planes: low half (bit planes 0-3) and high half (4-7) in separate arrays
  // so a warp's 16-byte accesses to consecutive words are bank-conflict free
  const int half = (P.R + 2 * n + 6) * P.nw_max * 4;
  uint32_t* skeys = reinterpret_cast<uint32_t*>(smem + P.sm_skeys);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P.sm_bar);

  const int slots = nrows * ccols;
  const bool local_keys = slots <= P.key_slots;

  // phase clock (stats runs): thread 0 keeps its stamps in shared memory, so
  // no register stays live across the kernel for them
  long long* stamps = reinterpret_cast<long long*>(smem + P.sm_bar + 16);
  if (STATS && P.phase_cycles && tid == 0) stamps[0] = clock64();
  // --- 1. stage the rows [ya, yb), columns [max(bx0,0), ...) of this tile
  if (k > 0 && P.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint8_t* frame = L.img + f * L.fstride;
  const int gx0 = max(bx0, 0);
  const int sx0 = gx0 - bx0;  // multiple of 16
  int row_bytes = min(bx0 + SW, L.pitch) - gx0;
  row_bytes = min(row_bytes, ((w + 15) & ~15) - gx0);
  if (L.tmap_ok) {
    // the stage's rows [iy0, iy0 + rows) x columns [bx0, bx0 + SW) of frame f
    // in one tensor copy (negative or past-the-edge coordinates read zeros)
    if (tid == 0) {
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = static_cast<uint32_t>(SW * (P.R + 2 * n + 6));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                   : "memory");
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&L.tmap)), "r"(bx0), "r"(iy0), "r"(f), "r"(b)
          : "memory");
    }
  } else if (L.tma) {
    row_bytes &= ~15;
    if (tid == 0) {
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = static_cast<uint32_t>(row_bytes * (yb - ya));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                   : "memory");
    }
  } else {
    for (int i = tid; i < (yb - ya) * row_bytes; i += kThreads) {
      const int y = ya + i / row_bytes, x = i % row_bytes;
      stage[(y - iy0) * SW + sx0 + x] = frame[static_cast<size_t>(y) * L.pitch + gx0 + x];
    }
  }
  if (local_keys) {
#pragma unroll 1
    for (int i = tid; i < slots; i += kThreads) skeys[i] = 0u;
  }
  // with the tensor copy, thread 0 armed the mbarrier and warp 0 alone polls
  // it: a warp-level sync suffices (the CTA barrier after the poll orders the
  // key clears); the per-row copies and the plain loads need the CTA barrier
  if (L.tmap_ok)
    __syncwarp();
  else
    __syncthreads();
  if (L.tma || L.tmap_ok) {
    // row copies (one per thread, the barrier is armed) unless the tensor
    // copy is in flight, then one warp waits for the transaction count
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    for (int y = ya + tid; !L.tmap_ok && y < yb; y += kThreads) {
      const uint32_t dst = static_cast<uint32_t>(
          __cvta_generic_to_shared(stage + (y - iy0) * SW + sx0));
      const uint8_t* src = frame + static_cast<size_t>(y) * L.pitch + gx0;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(dst), "l"(src), "r"(row_bytes), "r"(b)
          : "memory");
    }
    // one warp polls the transaction count (each poll is an issued
    // instruction sequence); the others wait at the CTA barrier, which
    // also orders the copied rows before their reads
#ifndef FLKB_WAIT_ALL
#define FLKB_WAIT_ALL 0
#endif
    if (FLKB_WAIT_ALL || warp == 0) {
      uint32_t done = 0;
      while (!done) {  // suspend hint: sleep in the barrier unit rather than re-issue
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(b), "r"(20000)
            : "memory");
      }
    }
    if (!FLKB_WAIT_ALL) __syncthreads();
  }

  // --- 1b. level-0 CTAs write pyramid levels 1 (and 2) of their own rows
  //         [y0, y1) x [x_lo, x_hi) from the staged rows: each thread turns a
  //         16x4 level-0 block into 8x2 level-1 and 4x1 level-2 pixels with the
  //         cascaded 2x2 round-half-up mean (image.cpp:50-62)
  if (k == 0 && P.pyr_levels > 0) {
    const int w1 = w >> 1, h1 = h >> 1, w2 = w1 >> 1, h2 = h1 >> 1;
    const int bxn = (x_hi - x_lo + 15) >> 4, byn = (y1 - y0 + 3) >> 2;
    const Level& L1 = P.lv[1];
    uint8_t* o1 = P.pyr_img[1] + f * L1.fstride;
    uint8_t* o2 = P.pyr_levels > 1 ? P.pyr_img[2] + f * P.lv[2].fstride : nullptr;
    const float inv_bxn = 1.0f / static_cast<float>(bxn);
    for (int i = tid; i < bxn * byn; i += kThreads) {
      // i / bxn: (i + 1/2) / bxn is at least 1/(2 bxn) from an integer, far
      // more than the float error for i < 2^16
      const int by = __float2int_rz((static_cast<float>(i) + 0.5f) * inv_bxn), bxi = i - by * bxn;
      const int x = x_lo + 16 * bxi, y = y0 + 4 * by;
      const uint8_t* sp = stage + (y - iy0) * SW + (x - bx0);
      const uint4 r0 = *reinterpret_cast<const uint4*>(sp);
      const uint4 r1 = *reinterpret_cast<const uint4*>(sp + SW);
      const uint4 r2 = *reinterpret_cast<const uint4*>(sp + 2 * SW);
      const uint4 r3 = *reinterpret_cast<const uint4*>(sp + 3 * SW);
      const uint32_t a0 = down4(r0.x, r0.y, r1.x, r1.y), a1 = down4(r0.z, r0.w, r1.z, r1.w);
      const uint32_t b0 = down4(r2.x, r2.y, r3.x, r3.y), b1 = down4(r2.z, r2.w, r3.z, r3.w);
      const int X1 = x >> 1, Y1 = y >> 1;
      auto put8 = [&](int yy, uint32_t lo, uint32_t hi) {
        if (yy >= h1) return;
        uint8_t* d = o1 + static_cast<size_t>(yy) * L1.pitch + X1;
        if (X1 + 8 <= w1) {
          *reinterpret_cast<uint2*>(d) = make_uint2(lo, hi);
        } else {
          for (int j = 0; X1 + j < w1; ++j)
            d[j] = static_cast<uint8_t>((j < 4 ? lo >> (8 * j) : hi >> (8 * (j - 4))) & 0xFFu);
        }
      };
      put8(Y1, a0, a1);
      put8(Y1 + 1, b0, b1);
      if (o2 && (y >> 2) < h2) {
        const int X2 = x >> 2;
        const uint32_t c = down4(a0, a1, b0, b1);
        uint8_t* d = o2 + static_cast<size_t>(y >> 2) * P.lv[2].pitch + X2;
        if (X2 + 4 <= w2) {
          *reinterpret_cast<uint32_t*>(d) = c;
        } else {
          for (int j = 0; X2 + j < w2; ++j) d[j] = static_cast<uint8_t>((c >> (8 * j)) & 0xFFu);
        }
      }
    }
  }

  // --- 2. bit planes of every staged row
  {
    const int tasks = (yb - ya) * nw;
    TaskIter it(tid, nw, L.div_nw);
    for (int t = tid; t < tasks; t += kThreads, it.next()) {
      const int r = ya - iy0 + it.row, j = it.j;
      const int bx = kOwn * j;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(stage + r * SW + (bx & ~3));
      uint32_t a[9], wv[8], pl[8];
#pragma unroll
      for (int i = 0; i < 9; ++i) a[i] = src[i];
      const uint32_t sel = (bx & 2) ? 0x5432u : 0x3210u;
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = __byte_perm(a[i], a[i + 1], sel);
      transpose32x8(wv, pl, P.pow2);
      uint32_t* dst = planes + (r * P.nw_max + j) * 4;
      *reinterpret_cast<uint4*>(dst) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
      *reinterpret_cast<uint4*>(dst + half) = make_uint4(pl[4], pl[5], pl[6], pl[7]);
    }
  }
  __syncthreads();

  // --- 3. bit-sliced corner masks for the FAST rows
  const int fast_rows = cy_hi - cy_lo;
  // Antipodal ring positions i, i + 8 (o_{i+8} = -o_i) give
  //   dark_i(p) = bright_{i+8}(p + o_i),  bright_i(p) = dark_{i+8}(p + o_i)
  // under the saturating thresholds sat(c -+ eps) (I(q) + eps < I(p) either
  // way), so only the 7 positions pointing down (dy > 0) and position 4 are
  // compared; the 7 pointing up are the down masks of the rows 1-3 above,
  // shifted by dx lanes, and position 12 is position 4 of the same row
  // shifted by 3 (fast.cpp:221-247 decides exactly the same). The CTA walks
  // its rows in waves of kThreads / nw rows (one (row, word) per thread):
  // pass A compares and publishes the down masks in a ring of wave + 3 rows,
  // pass B derives the up masks from the three rows above and runs the
  // segment tests. Rows cy_lo-3 .. cy_lo-1 only feed the rows below them.
  {
    const uint32_t (&E)[8] = P.emask;  // eps bit masks, constant-bank operands
    const int stride = P.nw_max * 4;
    const int wave = L.div_nw(kThreads);  // rows per wave
    const int ring = wave + 3;
    const int tr = L.div_nw(tid), j = tid - tr * nw;
    const bool lane_on = tr < wave;
    uint4* xv = reinterpret_cast<uint4*>(smem + P.sm_xrow);  // [4][ring][nw]
    const int vs = ring * nw;
    const int ytop = cy_lo - 3;
    int sbase = 0;  // ring slot of row w0
#pragma unroll 1
    for (int w0 = ytop; w0 < cy_hi; w0 += wave) {
      const int y = w0 + tr;
      const bool on = lane_on && y < cy_hi;
      int slot = sbase + tr;
      if (slot >= ring) slot -= ring;
      uint32_t dk[16], bk[16];
      if (on) {
        // pass A: clamped thresholds sat(c - eps), sat(c + eps) of row y,
        // then positions 4 (3,0), 5 (3,1), 11 (-3,1), 6 (2,2), 10 (-2,2),
        // 7 (1,3), 8 (0,3), 9 (-1,3)
        const uint32_t* pl = planes + j * 4 + (y - iy0) * stride;
        const uint32_t* ph = pl + half;
        auto load_planes = [&](int dy, uint32_t (&q)[8]) {
          const uint4 u = *reinterpret_cast<const uint4*>(pl + dy * stride);
          const uint4 v = *reinterpret_cast<const uint4*>(ph + dy * stride);
          q[0] = u.x; q[1] = u.y; q[2] = u.z; q[3] = u.w;
          q[4] = v.x; q[5] = v.y; q[6] = v.z; q[7] = v.w;
        };
        uint32_t c[8], lo[8], hi[8], br = 0, cy = 0;
        load_planes(0, c);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          // plain C so ptxas can take E[b] straight from the constant bank
          lo[b] = c[b] ^ E[b] ^ br;
          br = (~c[b] & E[b]) | (~c[b] & br) | (E[b] & br);
          hi[b] = c[b] ^ E[b] ^ cy;
          cy = (c[b] & E[b]) | (c[b] & cy) | (E[b] & cy);
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) {  // saturate: no ring byte is < 0 or > 255
          lo[b] &= ~br;
          hi[b] |= cy;
        }
#pragma unroll
        for (int dy = 0; dy <= 3; ++dy) {
          uint32_t q[8];
          if (dy == 0) {
#pragma unroll
            for (int b = 0; b < 8; ++b) q[b] = c[b];
          } else {
            load_planes(dy, q);
          }
#pragma unroll
          for (int i = 4; i <= 11; ++i) {
            if (ring_dy(i) != dy) continue;
            const int dx = ring_dx(i);
            uint32_t sh[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) sh[b] = shift_fma(q[b], dx, P.pow2);
            dk[i] = sliced_less(sh, lo);
            bk[i] = sliced_less(hi, sh);
          }
        }
        xv[slot * nw + j] = make_uint4(dk[5], dk[11], bk[5], bk[11]);
        xv[vs + slot * nw + j] = make_uint4(dk[6], dk[10], bk[6], bk[10]);
        xv[2 * vs + slot * nw + j] = make_uint4(dk[7], dk[8], dk[9], bk[7]);
        *reinterpret_cast<uint2*>(xv + 3 * vs + slot * nw + j) = make_uint2(bk[8], bk[9]);
      }
      __syncthreads();
      if (on && y >= cy_lo) {
        // pass B: the up positions from the rows above (ring slots y-1..y-3)
        const int s1 = slot >= 1 ? slot - 1 : slot - 1 + ring;
        const int s2 = slot >= 2 ? slot - 2 : slot - 2 + ring;
        const int s3 = slot >= 3 ? slot - 3 : slot - 3 + ring;
        const uint4 a = xv[s1 * nw + j];           // row y-1: dk5, dk11, bk5, bk11
        const uint4 b2 = xv[vs + s2 * nw + j];     // row y-2: dk6, dk10, bk6, bk10
        const uint4 c3 = xv[2 * vs + s3 * nw + j]; // row y-3: dk7, dk8, dk9, bk7
        const uint2 d3 = *reinterpret_cast<const uint2*>(xv + 3 * vs + s3 * nw + j);  // bk8, bk9
        dk[3] = shift_fma(a.w, 3, P.pow2);
        bk[3] = shift_fma(a.y, 3, P.pow2);
        dk[13] = shift_fma(a.z, -3, P.pow2);
        bk[13] = shift_fma(a.x, -3, P.pow2);
        dk[2] = shift_fma(b2.w, 2, P.pow2);
        bk[2] = shift_fma(b2.y, 2, P.pow2);
        dk[14] = shift_fma(b2.z, -2, P.pow2);
        bk[14] = shift_fma(b2.x, -2, P.pow2);
        dk[1] = shift_fma(d3.y, 1, P.pow2);
        bk[1] = shift_fma(c3.z, 1, P.pow2);
        dk[0] = d3.x;
        bk[0] = c3.y;
        dk[15] = shift_fma(c3.w, -1, P.pow2);
        bk[15] = shift_fma(c3.x, -1, P.pow2);
        dk[12] = shift_fma(bk[4], -3, P.pow2);
        bk[12] = shift_fma(dk[4], -3, P.pow2);
        // owned bits [3, 29) that fall inside the FAST columns
        const int xb = bx0 + kOwn * j;
        const int lo_b = max(3, cx_lo - xb), hi_b = min(29, cx_hi - xb);
        const uint32_t valid = hi_b > lo_b ? ((hi_b >= 32 ? 0xFFFFFFFFu : ((1u << hi_b) - 1u)) &
                                              ~((1u << lo_b) - 1u))
                                           : 0u;
        cm[(y - cy_lo) * nw + j] = sliced_corners<N>(dk, bk, valid);
      }
      sbase += wave;
      if (sbase >= ring) sbase -= ring;
      __syncthreads();  // the next wave reuses the ring; after the last, cm is complete
    }
  }

  // --- 4. one CTA-wide corner list (row-major task order) from a block scan
  //        of per-task corner counts; the score tile (aliasing the dead
  //        planes) is zeroed meanwhile. An entry is the corner's index in the
  //        score tile, (y - fy0) * RP + (x - x_lo + 2n): the tile store takes it
  //        as is, the stage address is one IMAD.HI + one IMAD away, and the
  //        order of entries is the (y, x) order the in-CTA keys rank by.
  const int tasks_f = max(fast_rows, 0) * nw;
  const int per = (tasks_f + kThreads - 1) / kThreads;
  const int tb = min(tid * per, tasks_f), te = min(tb + per, tasks_f);
  // List range of the suppressed rows [y0, y1): tasks [T0, T1) are row-major,
  // so their corners are entries [e_lo, e_hi); the owner of task T notes its
  // local offset while counting and records the list index after the scan.
  const int T0 = min(max(max(y0, 3) - cy_lo, 0) * nw, tasks_f);
  const int T1 = min(max(min(y1, h - 3) - cy_lo, 0) * nw, tasks_f);
  int cnt = 0, pre0 = -1, pre1 = -1;
  for (int t = tb; t < te; ++t) {
    if (t == T0) pre0 = cnt;
    if (t == T1) pre1 = cnt;
    cnt += __popc(cm[t]);
  }
  {
    uint4* z = reinterpret_cast<uint4*>(tile_s);
    const int n16 = ((P.R + 2 * n) * RP * 2) / 16;
    for (int i = tid; i < n16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) scan[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < kWarps ? scan[lane] : 0;
    int acc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, acc, o);
      if (lane >= o) acc += u;
    }
    if (lane < kWarps) scan[lane] = acc - v;
    if (lane == 31) scan[kWarps] = scan[kWarps + 1] = scan[kWarps + 2] = acc;
  }
  __syncthreads();
  const int base = scan[warp] + incl - cnt;  // this thread's first list index
  const int total = scan[kWarps];
  // (read after the scoring barrier)
  if (pre0 >= 0) scan[kWarps + 1] = base + pre0;
  if (pre1 >= 0) scan[kWarps + 2] = base + pre1;
  const int cap = P.cap;
  const int row_tb = L.div_nw(tb), j_tb = tb - row_tb * nw;
  // Score-tile column of stage column xs: xs + bx0 - (x_lo - 2n), i.e. an n-wide
  // zero margin left of the FAST columns.
  const int tcol = bx0 - (x_lo - 2 * n);
  // entry of bit 0 of task tb's word: tile row (row_tb + cy_lo - fy0), tile
  // column kOwn * j_tb + tcol; the next word of a row is kOwn further, a row
  // wrap adds RP - kOwn * nw
  const uint32_t eb_tb = static_cast<uint32_t>((row_tb + cy_lo - fy0) * RP + kOwn * j_tb + tcol);
  const uint32_t e_wrap = static_cast<uint32_t>(RP - kOwn * nw);
  // Writes the entries with list index in [w0, w0 + cap) to list[index - w0].
  auto build = [&](int w0) {
    if (total <= cap) {
      // Common case, every entry fits: per word slot, the warp either lets each
      // lane walk its own bits (cost ~ max popc) or expands the non-empty words
      // one at a time across the lanes (cost ~ non-empty words), whichever is
      // cheaper for this slot.
      int pos = base, j = j_tb;
      uint32_t e0 = eb_tb;
      for (int q = 0; q < per; ++q) {
        const int t = tb + q;
        uint32_t m = t < te ? cm[t] : 0u;
        const int c = __popc(m);
        const unsigned nz = __ballot_sync(0xffffffffu, m != 0u);
        const int mx = __reduce_max_sync(0xffffffffu, c);
        if (mx <= 2 * __popc(nz)) {
          // two bits per trip, lowest and highest, filling the word's entries
          // from both ends (the order inside a word is free: rounds and the
          // suppression range are word-granular); a lone last bit is written
          // twice to the same slot
          uint16_t* a = list + pos;
          uint16_t* z = list + pos + c - 1;
          while (m) {  // unrolled by two: up to four bits per trip
            // highest set bit hb (FLO), lowest (BREV + FLO.SH); both cleared
            uint32_t hb = bfind(m);
            a[0] = static_cast<uint16_t>(e0 + (__ffs(m) - 1));
            z[0] = static_cast<uint16_t>(e0 + hb);
            m &= (m - 1u) & ~bit(hb);
            if (!m) break;
            hb = bfind(m);
            a[1] = static_cast<uint16_t>(e0 + (__ffs(m) - 1));
            z[-1] = static_cast<uint16_t>(e0 + hb);
            m &= (m - 1u) & ~bit(hb);
            a += 2;
            z -= 2;
          }
        } else {
          unsigned z = nz;
          while (z) {
            const int src = __ffs(z) - 1;
            z &= z - 1;
            const uint32_t wv = __shfl_sync(0xffffffffu, m, src);
            const int p = __shfl_sync(0xffffffffu, pos, src);
            const uint32_t e = __shfl_sync(0xffffffffu, e0, src);
            if ((wv >> lane) & 1u)
              list[p + __popc(wv & ((1u << lane) - 1u))] = static_cast<uint16_t>(e + lane);
          }
        }
        pos += c;
        e0 += kOwn;
        if (++j == nw) {
          j = 0;
          e0 += e_wrap;
        }
      }
      return;
    }
    if (base >= w0 + cap || base + cnt <= w0) return;
    int pos = base, j = j_tb;
    uint32_t e0 = eb_tb;
    for (int t = tb; t < te; ++t) {
      uint32_t m = cm[t];
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        if (pos >= w0 && pos < w0 + cap) list[pos - w0] = static_cast<uint16_t>(e0 + b);
        ++pos;
      }
      e0 += kOwn;
      if (++j == nw) {
        j = 0;
        e0 += e_wrap;
      }
    }
  };
  // tile row of an entry: one IMAD.HI (exact for entries < 2^16)
  const uint32_t rp_magic = RADIUS == 1 ? kRpMagic1 : P.rp_magic;
  // stage byte of tile index 0's pixel: stage row 3 (tile row 0 = image row
  // fy0 = iy0 + 3), stage column -tcol; tile row r adds SW - RP on top of r * RP
  const uint8_t* const stage_e = stage + 3 * SW - tcol;
  const uint32_t list_s = static_cast<uint32_t>(__cvta_generic_to_shared(list));
  for (int w0 = 0; w0 < total; w0 += cap) {
    if (w0 > 0) __syncthreads();  // the previous round's entries are consumed
    build(w0);
    __syncthreads();
    const int m_end = min(cap, total - w0);
    // shared-address induction: one add per trip for the entry address and the bound
#pragma unroll kScoreUnroll
    for (uint32_t la = list_s + 2u * tid; la < list_s + 2u * m_end; la += 2u * kThreads) {
      const uint32_t ent = lds_u16(la);
      const uint32_t trow = __umulhi(ent, rp_magic);
      const uint8_t* sp = stage_e + mad_fma(trow, static_cast<uint32_t>(SW - RP), ent);
      const uint32_t cc = sp[0];
      int sc;
      if (KIND == kSadB) {
        uint32_t rb[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) rb[i] = sp[ring_dy(i) * SW + ring_dx(i)];
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)  // bytes packed with IMAD (FMA pipe; the ALU pipe is the busy one)
          pk[q] = mad_fma(rb[4 * q + 3], P.pow2[24],
                          mad_fma(rb[4 * q + 2], P.pow2[16], mad_fma(rb[4 * q + 1], P.pow2[8], rb[4 * q])));
        sc = sad_b_packed(pk, cc, static_cast<uint32_t>(P.eps), P.neg16eps);
      } else {
        int ring[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ring[i] = sp[ring_dy(i) * SW + ring_dx(i)];
        sc = fast_score<N, KIND>(static_cast<int>(cc), ring, P.eps);
      }
      tile_s[ent] = static_cast<uint16_t>(sc);
    }
  }
  __syncthreads();
  if (STATS && P.phase_cycles && tid == 0) stamps[1] = clock64();
  if (P.dbg_map) {  // diagnostic score dump (flkb_detector_fused_responses)
    uint16_t* out = P.dbg_map + f * P.dbg_fstride + L.dbg_off;
    const int tw = x_hi - x_lo;
    for (int i = tid; i < (y1 - y0) * tw; i += kThreads) {
      const int y = y0 + i / tw, x = x_lo + i % tw;
      out[static_cast<size_t>(y) * L.dbg_pitch + x] =
          static_cast<uint16_t>(tile_s[(y - fy0) * RP + (x - x_lo) + 2 * n] >> kTileShift);
    }
  }

  // --- 5. suppression + per-cell keys for the candidates in rows [y0, y1):
  //        a contiguous range of the list, since tasks are row-major
  unsigned long long n_cand = 0, n_cmp = 0;
  {
    // the tile's own columns [x_lo, x_hi) are tile columns [2n, 2n + span):
    // the list holds corners of FAST columns only, so one unsigned test on the
    // tile column drops the halo columns of the neighbouring tiles
    const unsigned tspan = static_cast<unsigned>(x_hi - x_lo);
    const int e_lo = T1 > T0 ? scan[kWarps + 1] : 0;
    const int e_hi = T1 > T0 ? scan[kWarps + 2] : 0;
    const int rp = RP;
    const int xo = x_lo - 2 * n;  // image x of tile column 0
    // cell map constants; the additive parts and the CTA's first cell row
    // fold into one base slot
    const uint32_t cmx = L.cmx, cmy = L.cmy;
    uint32_t* const kbase = skeys + static_cast<int>(L.ccy - static_cast<uint32_t>(cr0)) * ccols +
                            static_cast<int>(L.ccx) - cc0;
    const uint32_t kbase_s = static_cast<uint32_t>(__cvta_generic_to_shared(kbase));
    for (int w0 = e_lo; w0 < e_hi; w0 += cap) {
      const bool resident = total <= cap;  // the scoring list is still in place
      const int off = resident ? 0 : w0;
      if (!resident) {
        __syncthreads();
        build(w0);
        __syncthreads();
      }
      const int m_end = resident ? e_hi : min(w0 + cap, e_hi);
      // the loop is instantiated with and without the counters, so the
      // fast path carries no per-candidate stats test
      auto suppress = [&](auto local) {
        constexpr bool LOCAL = decltype(local)::value;
#pragma unroll kNmsUnroll
        for (uint32_t la = list_s + 2u * (w0 - off + tid); la < list_s + 2u * (m_end - off);
             la += 2u * kThreads) {
          const uint32_t ent = lds_u16(la);
          const uint32_t trow = __umulhi(ent, rp_magic);
          const uint32_t xcol = ent - trow * static_cast<uint32_t>(rp);
          if (xcol - static_cast<uint32_t>(2 * n) >= tspan) continue;  // halo column
          const uint16_t* row = tile_s + ent;
          const int s = row[0];
          // a corner whose score is 0 (MT, eps 0) is no candidate; a SAD score
          // sums >= N positive terms, so it is > 0 for every corner
          if (KIND == kMt && s == 0) continue;
          if constexpr (STATS) {
            bool keep = true;
            ++n_cand;
            uint32_t cmp = 0;
            const int x = xo + static_cast<int>(xcol), y = fy0 + static_cast<int>(trow);
            for (int rr = 1; rr <= n && keep; ++rr) {
              auto visit = [&](int dx, int dy) {
                if (!keep) return;
                const int nx = x + dx, ny = y + dy;
                if (nx < 0 || ny < 0 || nx >= w || ny >= h) return;
                ++cmp;
                const int v = row[dy * rp + dx];
                if (v > s || (v == s && (dy < 0 || (dy == 0 && dx < 0)))) keep = false;
              };
              for (int dx = -rr; dx <= rr; ++dx) visit(dx, -rr);
              for (int dy = -rr + 1; dy <= rr; ++dy) visit(rr, dy);
              for (int dx = rr - 1; dx >= -rr; --dx) visit(dx, rr);
              for (int dy = rr - 1; dy >= -rr + 1; --dy) visit(-rr, dy);
            }
            n_cmp += cmp;
            if (!keep) continue;
          } else if (RADIUS == 1) {
            // earlier neighbours must be strictly lower, later ones not higher;
            // out-of-image neighbours read the tile's zero margin
            const int e0 = max(max(row[-rp - 1], row[-rp]), max(row[-rp + 1], row[-1]));
            const int l0 = max(max(row[1], row[rp - 1]), max(row[rp], row[rp + 1]));
            if (e0 >= s || l0 > s) continue;
          } else {
            bool keep = true;
            for (int dy = -n; dy <= n && keep; ++dy)
              for (int dx = -n; dx <= n; ++dx) {
                const int v = row[dy * rp + dx];
                const bool earlier = dy < 0 || (dy == 0 && dx < 0);
                if (v > s || (v == s && earlier)) {
                  keep = false;
                  break;
                }
              }
            if (!keep) continue;
          }
          const uint32_t x = static_cast<uint32_t>(xo) + xcol, y = static_cast<uint32_t>(fy0) + trow;
          if (LOCAL) {
            // 32-bit key inside the CTA: score, then smaller y, then smaller x
            // (the level is fixed per CTA), as s << 16 | (0xFFFF - entry) --
            // entries ascend in (y, x) order; the cell with one IMAD.HI per
            // coordinate (no table loads)
            const uint32_t key = mad_fma(static_cast<uint32_t>(s), P.pow2[16 - kTileShift], ent ^ 0xFFFFu);
            const uint32_t cx = __umulhi(x, cmx);
            const uint32_t cy = __umulhi(y, cmy);
            // shared byte address of the slot: one IMAD for cy * ccols + cx, one
            // LEA onto the CTA's (uniform) key base
            const uint32_t addr = kbase_s + 4u * mad_fma(cy, static_cast<uint32_t>(ccols), cx);
            asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(addr), "r"(key) : "memory");
          } else {
            const int X = static_cast<int>(x) << k, Y = static_cast<int>(y) << k;
            atomicMax(P.keys + static_cast<size_t>(f) * P.cells + P.div_ch(Y) * P.cols + P.div_cw(X),
                      pack_key(s >> kTileShift, k, X, Y));
          }
        }
      };
#if FLKB_KEYS
      // A/B variant: the warp combines its
      // survivors' 32-bit keys before the shared atomics -- FLKB_KEYS=1 groups
      // lanes by cell (match.any + redux.max, one ATOMS.MAX per distinct cell
      // of the warp), FLKB_KEYS=2 is the paper's shfl_xor butterfly over
      // packed keys when every survivor of the warp falls in one cell
      // (per-lane atomics otherwise). Radius 1, shared keys, no counters.
      if (!STATS && RADIUS == 1 && local_keys) {
        for (int eb = w0 + warp * 32; eb < m_end; eb += kThreads) {  // warp-uniform trips
          const int e = eb + lane;
          uint32_t key = 0;
          int slot = -1;
          if (e < m_end) {
            const uint32_t ent = list[e - off];
            const uint32_t trow = __umulhi(ent, rp_magic);
            const uint32_t xcol = ent - trow * static_cast<uint32_t>(rp);
            const uint16_t* row = tile_s + ent;
            const int sc = row[0];
            const int e0 = max(max(row[-rp - 1], row[-rp]), max(row[-rp + 1], row[-1]));
            const int l0 = max(max(row[1], row[rp - 1]), max(row[rp], row[rp + 1]));
            if (xcol - static_cast<uint32_t>(2 * n) < tspan && sc != 0 && e0 < sc && l0 <= sc) {
              const uint32_t x = static_cast<uint32_t>(xo) + xcol, y = static_cast<uint32_t>(fy0) + trow;
              key = mad_fma(static_cast<uint32_t>(sc), P.pow2[16 - kTileShift], ent ^ 0xFFFFu);
              slot = static_cast<int>(mad_fma(__umulhi(y, cmy), static_cast<uint32_t>(ccols), __umulhi(x, cmx)));
            }
          }
#if FLKB_KEYS == 1
          const unsigned grp = __match_any_sync(0xffffffffu, slot);
          const uint32_t kmax = __reduce_max_sync(grp, key);
          if (slot >= 0 && lane == __ffs(grp) - 1) atomicMax(kbase + slot, kmax);
#else
          const int s0 = __shfl_sync(0xffffffffu, slot, __ffs(__ballot_sync(0xffffffffu, slot >= 0)) - 1);
          if (__all_sync(0xffffffffu, slot < 0 || slot == s0)) {
            uint32_t k = key;
#pragma unroll
            for (int o = 16; o; o >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, o));
            if (lane == 0 && k) atomicMax(kbase + s0, k);
          } else if (slot >= 0) {
            atomicMax(kbase + slot, key);
          }
#endif
        }
      } else
#endif
      if (local_keys)
        suppress(std::true_type{});
      else
        suppress(std::false_type{});
      if (resident) break;
    }
  }
  if (STATS) {
    for (int o = 16; o; o >>= 1) {
      n_cand += __shfl_xor_sync(0xffffffffu, n_cand, o);
      n_cmp += __shfl_xor_sync(0xffffffffu, n_cmp, o);
    }
    if (lane == 0 && (n_cand | n_cmp)) {
      atomicAdd(P.stats + 2 * f, n_cand);
      atomicAdd(P.stats + 2 * f + 1, n_cmp);
    }
  }
  // phase clock (stats runs only)
  auto phase_end = [&] {
    if (STATS && P.phase_cycles && tid == 0) {
      const long long t_end = clock64();
      atomicAdd(P.phase_cycles, static_cast<unsigned long long>(stamps[1] - stamps[0]));
      atomicAdd(P.phase_cycles + 1, static_cast<unsigned long long>(t_end - stamps[1]));
    }
  };
  if (!local_keys) {
    phase_end();
    return;
  }
  __syncthreads();

  // --- 6. flush the shared cell keys into the frame's global keys
  const float inv_cc = 1.0f / static_cast<float>(ccols);
#pragma unroll 1
  for (int i = tid; i < slots; i += kThreads) {
    const uint32_t key = skeys[i];
    if (!key) continue;
    // slot row i / ccols: (i + 1/2) / ccols is at least 1/(2 ccols) from an
    // integer, far more than the float error for i < 2^16
    const int rr = __float2int_rz((static_cast<float>(i) + 0.5f) * inv_cc);
    const uint32_t ent = (key & 0xFFFFu) ^ 0xFFFFu;  // the winner's tile index
    const uint32_t trow = __umulhi(ent, rp_magic);
    const int y = fy0 + static_cast<int>(trow);
    const int x = x_lo - 2 * n + static_cast<int>(ent - trow * static_cast<uint32_t>(RP));
    atomicMax(P.keys + static_cast<size_t>(f) * P.cells + (cr0 + rr) * P.cols + cc0 + (i - rr * ccols),
              pack_key(static_cast<int>(key >> 16), k, x << k, y << k));
  }
  phase_end();
}

}  // namespace fused
}  // namespace flkb
