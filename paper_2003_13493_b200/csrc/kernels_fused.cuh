// Fused FAST + score + window-max suppression + cell selection. sm_100a.
//
// One CTA walks down one column segment of one level of one frame in bands of
// R rows, carrying the halo (image rows, bit planes, corner masks, scores) of
// band b into band b+1, so no row is staged, sliced, tested or scored twice.
// Per band:
//
//  A. TMA   one elected thread issues cp.async.bulk row copies of the band's
//           new image rows into shared memory (mbarrier completion); the halo
//           rows were shifted up from the previous band.
//  B. SLICE every 32-byte window (stride 26 px) of a new row is transposed
//           into 8 bit planes: bit b of plane k = bit k of pixel x0+b. A word
//           "owns" its middle 26 pixels, so every ring offset (|dx| <= 3)
//           stays inside the word -- no neighbour exchange.
//  C. MASKS bit-sliced FAST on the new rows: thresholds L = sat(c-eps),
//           H = sat(c+eps) as planes; each of the 16 ring positions' shifted
//           planes (shifts issued as IMAD) compared by a one-LOP3-per-bit
//           borrow chain: dark_i = R_i < L, bright_i = H < R_i, 32 pixels per
//           instruction; the segment test is a sliding AND over the 16
//           position words. Identical to the reference LUT test
//           (fast.cpp:34-65, 221-247) for every mask and N.
//  D. LIST  a block scan of per-word corner counts (rows y0-n .. y1+n) builds
//           one CTA-wide corner list in row-major order (per-lane or
//           warp-cooperative expansion, whichever is cheaper per slot).
//  E. SCORE the new rows' corners (a contiguous list range): SAD-B through
//           VABSDIFF4 on packed ring bytes, SAD-A / MT through the register
//           forms of fast_math.cuh, into a zero-margin u16 score tile.
//  F. NMS   the band's own rows (another contiguous range) against the
//           (2n+1)^2 window with spiral_is_local_max's tie rule
//           (nms.cpp:48-79); survivors ATOMS.MAX a 32-bit in-cell key
//           (score, -y, -x inside the cell; level fixed per CTA) built from
//           per-column / per-row lookup tables.
//  G. FLUSH each non-empty cell key becomes the global u64 key (score,
//           -level, -y0, -x0) with one atomicMax -- the cross-level
//           cell_candidate_wins order (nms.cpp:41-46).
#pragma once

#include <cstdint>

#include "fused_prims.cuh"

namespace flkb {
namespace fused {

constexpr int kOwn = 26;  // pixels owned by one 32-bit plane word
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef FLKB_MIN_BLOCKS
#define FLKB_MIN_BLOCKS 3
#endif
constexpr int kMinBlocks = FLKB_MIN_BLOCKS;  // CTAs per SM the register budget targets
constexpr int kMaxLv = 16;

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
  const uint8_t* img;  // frame 0, row 0
  size_t fstride;
  int pitch, w, h;
  int tiles_x, tile_w;  // column tiles and NMS columns per tile
  int segs, seg_rows;   // row segments per column and rows per segment (multiple of R)
  int cta0;             // first blockIdx.x of this level
  int tma;              // rows may be fetched with cp.async.bulk
  int nw;               // plane words per row (max over the level's tiles)
  FastDiv div_nw, div_tiles;
};

struct Params {
  Level lv[kMaxLv];
  int levels;
  int eps, radius, R;
  int cell_w, cell_h, cols, cells;
  FastDiv div_cw, div_ch;
  int sw;         // stage row pitch (bytes)
  int nw_max;     // plane words per row, max over levels
  int rp;         // score tile pitch (u16)
  int key_slots;  // shared cell-key capacity per band
  int list_cap;   // corner-list capacity (u16 entries)
  unsigned long long* keys;
  unsigned long long* stats;
  uint32_t pow2[32];  // 1 << i, from the constant bank so shifts can issue as IMAD
};

struct Smem {
  int stage, planes, tile, cm, list, scan, skeys, colkey, rowkey, bar, total;
};

__host__ __device__ inline Smem smem_layout(const Params& p) {
  const int img_rows = p.R + 2 * p.radius + 6;
  const int fast_rows = p.R + 2 * p.radius;
  Smem s;
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) & ~(align - 1);
    const int at = off;
    off += bytes;
    return at;
  };
  s.stage = take(img_rows * p.sw, 128);
  s.planes = take(img_rows * p.nw_max * 32, 128);  // [2 halves][img_rows][nw_max][4 planes]
  s.tile = take(fast_rows * p.rp * 2, 16);
  s.cm = take(fast_rows * p.nw_max * 4, 16);
  s.list = take(p.list_cap * 2, 16);
  s.scan = take((kWarps + 8) * 4, 16);
  s.skeys = take(p.key_slots * 4, 16);
  s.colkey = take(p.sw * 4, 16);
  s.rowkey = take(fast_rows * 4, 16);
  s.bar = take(16, 16);
  s.total = off;
  return s;
}

__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {  // bits [lo, hi) of a word
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (hi <= lo) return 0u;
  return (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
}

template <int N, int KIND, int RADIUS>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_detect(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Smem S = smem_layout(P);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // --- which level, segment and column tile
  int k = 0;
  while (k + 1 < P.levels && static_cast<int>(blockIdx.x) >= P.lv[k + 1].cta0) ++k;
  const Level& L = P.lv[k];
  const int local = blockIdx.x - L.cta0;
  const int seg = L.div_tiles(local), tile = local - seg * L.tiles_x;
  const int f = blockIdx.y;
  const int n = RADIUS > 0 ? RADIUS : P.radius, w = L.w, h = L.h, R = P.R;
  const int s0 = seg * L.seg_rows, s1 = min(s0 + L.seg_rows, h);
  const int x_lo = tile * L.tile_w, x_hi = min(x_lo + L.tile_w, w);
  const int bx0 = (x_lo - n - 3) & ~15;  // stage column 0 <-> image x bx0
  const int nw = L.nw;
  const int cx_lo = max(x_lo - n, 3), cx_hi = min(x_hi + n, w - 3);  // FAST columns
  const int nx_lo = max(x_lo, 3), nx_hi = min(x_hi, w - 3);          // suppressed columns
  const int img_rows = R + 2 * n + 6, fast_rows = R + 2 * n;
  const int half = img_rows * P.nw_max * 4;
  const int tcol = bx0 - (x_lo - 2 * n);  // score-tile column of stage column xs: xs + tcol

  uint8_t* stage = smem + S.stage;
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + S.planes);
  uint16_t* tile_s = reinterpret_cast<uint16_t*>(smem + S.tile);
  uint32_t* cm = reinterpret_cast<uint32_t*>(smem + S.cm);
  uint16_t* list = reinterpret_cast<uint16_t*>(smem + S.list);
  int* scan = reinterpret_cast<int*>(smem + S.scan);
  uint32_t* skeys = reinterpret_cast<uint32_t*>(smem + S.skeys);
  uint32_t* colkey = reinterpret_cast<uint32_t*>(smem + S.colkey);
  uint32_t* rowkey = reinterpret_cast<uint32_t*>(smem + S.rowkey);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S.bar);
  const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(bar));

  const uint8_t* frame = L.img + f * L.fstride;
  const int gx0 = max(bx0, 0);
  const int sx0 = gx0 - bx0;  // multiple of 16
  const int row_bytes =
      (min(min(bx0 + P.sw, L.pitch), (w + 15) & ~15) - gx0) & (L.tma ? ~15 : ~0);

  // In-cell key part of every stage column: cell_x << 10 | (1023 - local x).
  const bool local_keys = P.key_slots > 0;
  if (local_keys) {
    for (int xs = tid; xs < P.sw; xs += kThreads) {
      const int x = max(bx0 + xs, 0);
      const int ccx = P.div_cw(x << k);
      const int ox = (ccx * P.cell_w + (1 << k) - 1) >> k;
      colkey[xs] = (static_cast<uint32_t>(ccx) << 10) | ((1023u - (x - ox)) & 1023u);
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase = 0;
  uint32_t E[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) E[b] = ((P.eps >> b) & 1) ? 0xFFFFFFFFu : 0u;
  unsigned long long n_cand = 0, n_cmp = 0;
  (void)lane;

  for (int y0 = s0; y0 < s1; y0 += R) {
    const bool first = y0 == s0;
    const int y1 = min(y0 + R, s1);
    const int iy0 = y0 - n - 3;  // stage row 0 <-> image row iy0
    const int fy0 = y0 - n;      // tile / cm row 0 <-> image row fy0
    // rows this band adds: image rows [na, nb), FAST rows [fa, fb)
    const int na = max(first ? iy0 : y0 + n + 3, 0), nb = min(y1 + n + 3, h);
    const int fa = first ? fy0 : y0 + n, fb = y1 + n;

    // --- A. shift the previous band's halo up by R rows, then fetch new rows
    __syncthreads();  // everyone is done with the previous band
    if (!first) {
      const int keep = 2 * n + 6;  // halo image rows (R >= keep: no overlap)
      {
        const uint4* src = reinterpret_cast<const uint4*>(stage + R * P.sw);
        uint4* dst = reinterpret_cast<uint4*>(stage);
        for (int i = tid; i < keep * P.sw / 16; i += kThreads) dst[i] = src[i];
      }
      for (int hh = 0; hh < 2; ++hh) {
        const uint4* src = reinterpret_cast<const uint4*>(planes + hh * half + R * P.nw_max * 4);
        uint4* dst = reinterpret_cast<uint4*>(planes + hh * half);
        for (int i = tid; i < keep * P.nw_max; i += kThreads) dst[i] = src[i];
      }
      {
        const uint4* src = reinterpret_cast<const uint4*>(tile_s + R * P.rp);
        uint4* dst = reinterpret_cast<uint4*>(tile_s);
        for (int i = tid; i < 2 * n * P.rp / 8; i += kThreads) dst[i] = src[i];
      }
      for (int i = tid; i < 2 * n * nw; i += kThreads) cm[i] = cm[R * nw + i];
      __syncthreads();
    }
    {  // zero the score-tile rows the new corners land in
      uint4* z = reinterpret_cast<uint4*>(tile_s + (fa - fy0) * P.rp);
      const int n16 = (fast_rows - (fa - fy0)) * P.rp / 8;
      for (int i = tid; i < n16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
    }
    if (local_keys) {
      for (int i = tid; i < P.key_slots; i += kThreads) skeys[i] = 0u;
      for (int r = tid; r < y1 - y0; r += kThreads) {  // own rows' in-cell row keys
        const int y = y0 + r;
        const int ccy = P.div_ch(y << k);
        const int oy = (ccy * P.cell_h + (1 << k) - 1) >> k;
        rowkey[r] = (static_cast<uint32_t>((ccy - P.div_ch(y0 << k)) * P.cols) << 10) |
                    ((1023u - (y - oy)) & 1023u);
      }
    }
    if (L.tma) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = static_cast<uint32_t>(row_bytes * max(nb - na, 0));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s),
                     "r"(bytes)
                     : "memory");
        for (int y = na; y < nb; ++y) {
          const uint32_t dst = static_cast<uint32_t>(
              __cvta_generic_to_shared(stage + (y - iy0) * P.sw + sx0));
          const uint8_t* src = frame + static_cast<size_t>(y) * L.pitch + gx0;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                  "r"(dst), "l"(src), "r"(row_bytes), "r"(bar_s)
              : "memory");
        }
      }
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar_s), "r"(phase)
            : "memory");
      }
      phase ^= 1u;
    } else {
      for (int i = tid; i < max(nb - na, 0) * row_bytes; i += kThreads) {
        const int y = na + i / row_bytes, x = i % row_bytes;
        stage[(y - iy0) * P.sw + sx0 + x] = frame[static_cast<size_t>(y) * L.pitch + gx0 + x];
      }
    }
    __syncthreads();

    // --- B. bit planes of the new rows
    {
      const int rows = max(nb - na, 0), tasks = rows * nw;
      int row = L.div_nw(tid), j = tid - row * nw;
      const int drow = L.div_nw(kThreads), dj = kThreads - drow * nw;
      for (int t = tid; t < tasks; t += kThreads) {
        const int r = na - iy0 + row;
        const int bx = kOwn * j;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(stage + r * P.sw + (bx & ~3));
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
        row += drow;
        j += dj;
        if (j >= nw) {
          j -= nw;
          ++row;
        }
      }
    }
    __syncthreads();

    // --- C. bit-sliced corner masks of the new FAST rows (0 outside [3, h-3))
    {
      const int tasks = (fb - fa) * nw;
      int row = L.div_nw(tid), j = tid - row * nw;
      const int drow = L.div_nw(kThreads), dj = kThreads - drow * nw;
      for (int t = tid; t < tasks; t += kThreads) {
        const int y = fa + row;
        uint32_t corner = 0u;
        if (y >= 3 && y < h - 3) {
          const int r = y - iy0;
          const uint32_t* base = planes + j * 4;
          auto row_planes = [&](int rr, uint32_t (&q)[8]) {
            const uint32_t* q4 = base + rr * P.nw_max * 4;
            const uint4 u = *reinterpret_cast<const uint4*>(q4);
            const uint4 v = *reinterpret_cast<const uint4*>(q4 + half);
            q[0] = u.x; q[1] = u.y; q[2] = u.z; q[3] = u.w;
            q[4] = v.x; q[5] = v.y; q[6] = v.z; q[7] = v.w;
          };
          uint32_t c[8], lo[8], hi[8];
          row_planes(r, c);
          {
            uint32_t br = 0, cy = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              lo[b] = lop3_xor3(c[b], E[b], br);
              br = lop3_maj_na(c[b], E[b], br);
              hi[b] = lop3_xor3(c[b], E[b], cy);
              cy = lop3_maj(c[b], E[b], cy);
            }
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              lo[b] &= ~br;  // c - eps < 0   -> 0
              hi[b] |= cy;   // c + eps > 255 -> 255
            }
          }
          uint32_t dk[16], bk[16];
#pragma unroll
          for (int dy = -3; dy <= 3; ++dy) {
            uint32_t q[8];
            row_planes(r + dy, q);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (ring_dy(i) != dy) continue;
              const int dx = ring_dx(i);
              uint32_t s[8];
#pragma unroll
              for (int b = 0; b < 8; ++b) s[b] = shift_fma(q[b], dx, P.pow2);
              dk[i] = sliced_less(s, lo);
              bk[i] = sliced_less(hi, s);
            }
          }
          const int xb = bx0 + kOwn * j;
          corner = (sliced_arc<N>(dk) | sliced_arc<N>(bk)) &
                   bit_range(max(3, cx_lo - xb), min(29, cx_hi - xb));
        }
        cm[(y - fy0) * nw + j] = corner;
        row += drow;
        j += dj;
        if (j >= nw) {
          j -= nw;
          ++row;
        }
      }
    }
    __syncthreads();

    // --- D. corner list over the FAST rows [fy0, y1 + n): block scan of
    //        per-task counts; entries (tile row << 10 | stage column)
    const int tasks_f = (fb - fy0) * nw;
    const int per = (tasks_f + kThreads - 1) / kThreads;
    const int tb = min(tid * per, tasks_f), te = min(tb + per, tasks_f);
    int cnt = 0;
    for (int t = tb; t < te; ++t) cnt += __popc(cm[t]);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) scan[warp] = incl;
    // list indices of three task boundaries: new FAST rows, own rows begin / end
    const int T_new = (fa - fy0) * nw;
    const int T_a = (max(y0, 3) - fy0) * nw, T_b = (max(min(y1, h - 3), max(y0, 3)) - fy0) * nw;
    if (tid == 0) scan[kWarps + 1] = scan[kWarps + 2] = scan[kWarps + 3] = -1;
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
      if (lane == 31) scan[kWarps] = acc;
    }
    __syncthreads();
    const int base = scan[warp] + incl - cnt;
    const int total = scan[kWarps];
    if (tb < te) {
      int pos = base;
      for (int t = tb; t < te; ++t) {
        if (t == T_new) scan[kWarps + 1] = pos;
        if (t == T_a) scan[kWarps + 2] = pos;
        if (t == T_b) scan[kWarps + 3] = pos;
        pos += __popc(cm[t]);
      }
    }
    const int cap = P.list_cap;
    const int row_tb = L.div_nw(tb), j_tb = tb - row_tb * nw;
    // Writes the entries with list index in [w0, w0 + cap) to list[index - w0].
    auto build = [&](int w0) {
      if (total <= cap) {
        // every entry fits: per word slot, the warp either lets each lane walk
        // its own bits (cost ~ max popc) or expands the non-empty words one at
        // a time across the lanes (cost ~ non-empty words), whichever is cheaper
        int pos = base, row = row_tb, j = j_tb;
        for (int q = 0; q < per; ++q) {
          const int t = tb + q;
          uint32_t m = t < te ? cm[t] : 0u;
          const uint32_t e0 = (static_cast<uint32_t>(row) << 10) | static_cast<uint32_t>(kOwn * j);
          const int c = __popc(m);
          const unsigned nz = __ballot_sync(0xffffffffu, m != 0u);
          const int mx = __reduce_max_sync(0xffffffffu, c);
          if (2 * mx <= 3 * __popc(nz)) {
            int p = pos;
            while (m) {
              const int b = __ffs(m) - 1;
              m &= m - 1;
              list[p++] = static_cast<uint16_t>(e0 + b);
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
          if (++j == nw) {
            j = 0;
            ++row;
          }
        }
        return;
      }
      if (base >= w0 + cap || base + cnt <= w0) return;
      int pos = base, row = row_tb, j = j_tb;
      for (int t = tb; t < te; ++t) {
        uint32_t m = cm[t];
        const uint32_t e0 = (static_cast<uint32_t>(row) << 10) | static_cast<uint32_t>(kOwn * j);
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          if (pos >= w0 && pos < w0 + cap) list[pos - w0] = static_cast<uint16_t>(e0 + b);
          ++pos;
        }
        if (++j == nw) {
          j = 0;
          ++row;
        }
      }
    };
    __syncthreads();
    const int e_new = scan[kWarps + 1] < 0 ? total : scan[kWarps + 1];
    const int e_a = scan[kWarps + 2] < 0 ? total : scan[kWarps + 2];
    const int e_b = scan[kWarps + 3] < 0 ? total : scan[kWarps + 3];
    const bool resident = total <= cap;
    if (resident) {
      build(0);
      __syncthreads();
    }

    // --- E. score the new rows' corners
    for (int w0 = e_new; w0 < total; w0 += cap) {
      if (!resident) {
        __syncthreads();
        build(w0);
        __syncthreads();
      }
      const int off = resident ? 0 : w0;
      const int m_end = resident ? total : min(w0 + cap, total);
      for (int e = w0 + tid; e < m_end; e += kThreads) {
        const int ent = list[e - off];
        const int tr = ent >> 10, xs = ent & 1023;
        const uint8_t* sp = stage + (tr + 3) * P.sw + xs;  // tile row tr = stage row tr + 3
        const uint32_t cc = sp[0];
        int sc;
        if (KIND == kSadB) {
          uint32_t rb[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) rb[i] = sp[ring_dy(i) * P.sw + ring_dx(i)];
          uint32_t pk[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            pk[q] = __byte_perm(__byte_perm(rb[4 * q], rb[4 * q + 1], 0x0040),
                                __byte_perm(rb[4 * q + 2], rb[4 * q + 3], 0x0040), 0x5410);
          sc = sad_b_packed(pk, cc, static_cast<uint32_t>(P.eps));
        } else {
          int ring[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) ring[i] = sp[ring_dy(i) * P.sw + ring_dx(i)];
          sc = fast_score<N, KIND>(static_cast<int>(cc), ring, P.eps);
        }
        tile_s[tr * P.rp + xs + tcol] = static_cast<uint16_t>(sc);
      }
      if (resident) break;
    }
    __syncthreads();

    // --- F. suppression + in-cell keys for the candidates of rows [y0, y1)
    {
      const int rp = P.rp;
      const int cr0 = P.div_ch(y0 << k);
      for (int w0 = e_a; w0 < e_b; w0 += cap) {
        if (!resident) {
          __syncthreads();
          build(w0);
          __syncthreads();
        }
        const int off = resident ? 0 : w0;
        const int m_end = resident ? e_b : min(w0 + cap, e_b);
        for (int e = w0 + tid; e < m_end; e += kThreads) {
          const int ent = list[e - off];
          const int tr = ent >> 10, xs = ent & 1023;
          const int x = bx0 + xs, y = fy0 + tr;
          if (x < nx_lo || x >= nx_hi) continue;  // a neighbouring tile's column
          const uint16_t* row = tile_s + tr * rp + xs + tcol;
          const int s = row[0];
          if (s == 0) continue;  // a corner whose score is 0 (MT, eps 0) is no candidate
          bool keep = true;
          if (P.stats) {
            ++n_cand;
            uint32_t cmp = 0;
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
          } else if (RADIUS == 1) {
            // earlier neighbours must be strictly lower, later ones not higher;
            // out-of-image neighbours read the tile's zero margin
            const int e0 = max(max(row[-rp - 1], row[-rp]), max(row[-rp + 1], row[-1]));
            const int l0 = max(max(row[1], row[rp - 1]), max(row[rp], row[rp + 1]));
            keep = e0 < s && l0 <= s;
          } else {
            for (int dy = -n; dy <= n && keep; ++dy)
              for (int dx = -n; dx <= n; ++dx) {
                const int v = row[dy * rp + dx];
                const bool earlier = dy < 0 || (dy == 0 && dx < 0);
                if (v > s || (v == s && earlier)) {
                  keep = false;
                  break;
                }
              }
          }
          if (!keep) continue;
          if (local_keys) {
            const uint32_t ck = colkey[xs], rk = rowkey[y - y0];
            const uint32_t key =
                (static_cast<uint32_t>(s) << 20) | ((rk & 1023u) << 10) | (ck & 1023u);
            atomicMax(skeys + (rk >> 10) + (ck >> 10), key);
          } else {
            const int X = x << k, Y = y << k;
            atomicMax(P.keys + static_cast<size_t>(f) * P.cells + P.div_ch(Y) * P.cols + P.div_cw(X),
                      pack_key(s, k, X, Y));
          }
        }
        if (resident) break;
      }

      // --- G. flush the band's cell keys into the frame's global keys
      if (local_keys) {
        __syncthreads();
        const int cr1 = P.div_ch((y1 - 1) << k);
        const int slots = (cr1 - cr0 + 1) * P.cols;
        for (int i = tid; i < slots; i += kThreads) {
          const uint32_t key = skeys[i];
          if (!key) continue;
          const int ccy = cr0 + i / P.cols, ccx = i - (i / P.cols) * P.cols;
          const int ox = (ccx * P.cell_w + (1 << k) - 1) >> k;
          const int oy = (ccy * P.cell_h + (1 << k) - 1) >> k;
          const int y = oy + 1023 - static_cast<int>((key >> 10) & 1023u);
          const int x = ox + 1023 - static_cast<int>(key & 1023u);
          atomicMax(P.keys + static_cast<size_t>(f) * P.cells + cr0 * P.cols + i,
                    pack_key(static_cast<int>(key >> 20), k, x << k, y << k));
        }
      }
    }
  }

  if (P.stats) {
    for (int o = 16; o; o >>= 1) {
      n_cand += __shfl_xor_sync(0xffffffffu, n_cand, o);
      n_cmp += __shfl_xor_sync(0xffffffffu, n_cmp, o);
    }
    if (lane == 0 && (n_cand | n_cmp)) {
      atomicAdd(P.stats + 2 * f, n_cand);
      atomicAdd(P.stats + 2 * f + 1, n_cmp);
    }
  }
}

}  // namespace fused
}  // namespace flkb
