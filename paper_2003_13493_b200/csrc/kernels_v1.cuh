// Staged sm_100a kernels: pyramid -> FAST score maps -> window-max + cell
// key reduction -> ballot compaction. One launch per stage and level.
//
// Semantics (bit-exact with the reference):
//   pyramid   L_k = (2x2 sum of L_{k-1} + 2) >> 2, cascaded (image.cpp:49-62)
//   FAST      score_at (fast.cpp:221-247) for 3 <= x < w-3, 3 <= y < h-3
//   NMS       spiral_is_local_max's survival rule (nms.cpp:48-79)
//   select    cell_candidate_wins's order (nms.cpp:41-46) as a u64 max
//   flatten   row-major non-empty cells (capi.cpp:260-269)
#pragma once

#include <cstdint>

#include "fast_math.cuh"

namespace flkb {

// --------------------------------------------------------------- pyramid

// One thread per 8 output pixels of level k from level k-1; 16-B row loads
// when aligned, byte loads at the ragged right edge.
__global__ void __launch_bounds__(256) k_pyramid_down(const uint8_t* __restrict__ src,
                                                      int spitch, size_t sfs,
                                                      uint8_t* __restrict__ dst, int dpitch,
                                                      size_t dfs, int wd, int hd, int vec_ok) {
  // a programmatic dependent (the fused detector) may launch now; its CTAs
  // that read the pyramid wait for this grid with griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  const int f = blockIdx.z;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x8 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (y >= hd || x8 >= wd) return;
  const uint8_t* r0 = src + f * sfs + static_cast<size_t>(2 * y) * spitch + 2 * x8;
  const uint8_t* r1 = r0 + spitch;
  uint8_t* out = dst + f * dfs + static_cast<size_t>(y) * dpitch + x8;
  if (vec_ok && x8 + 8 <= wd) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(r0));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(r1));
    uint2 o;
    o.x = down4(a.x, a.y, b.x, b.y);
    o.y = down4(a.z, a.w, b.z, b.w);
    *reinterpret_cast<uint2*>(out) = o;
  } else {
    const int n = min(8, wd - x8);
    for (int j = 0; j < n; ++j)
      out[j] = static_cast<uint8_t>((r0[2 * j] + r0[2 * j + 1] + r1[2 * j] + r1[2 * j + 1] + 2) >> 2);
  }
}

// Levels k and k+1 from level k-1 in one pass: one thread per 16x4 block of
// the source, 8x2 level-k pixels and 4x1 level-(k+1) pixels, cascaded
// (image.cpp:50-62: level k+1 is the mean of the rounded level-k pixels).
__global__ void __launch_bounds__(256) k_pyramid_down2(const uint8_t* __restrict__ src,
                                                       int spitch, size_t sfs,
                                                       uint8_t* __restrict__ d1, int p1,
                                                       uint8_t* __restrict__ d2, int p2, size_t dfs,
                                                       int w1, int h1, int w2, int h2, int vec_ok) {
  asm volatile("griddepcontrol.launch_dependents;");  // see k_pyramid_down
  const int f = blockIdx.z;
  const int ty = blockIdx.y * blockDim.y + threadIdx.y;     // level-k row pair, level-(k+1) row
  const int x8 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;  // first level-k column
  if (2 * ty >= h1 || x8 >= w1) return;
  const uint8_t* s0 = src + f * sfs + static_cast<size_t>(4 * ty) * spitch + 2 * x8;
  uint8_t* o1 = d1 + f * dfs + static_cast<size_t>(2 * ty) * p1 + x8;
  const bool two_rows = 2 * ty + 1 < h1;
  uint32_t a0, a1, b0 = 0, b1 = 0;
  if (vec_ok && x8 + 8 <= w1 && two_rows) {
    const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(s0));
    const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(s0 + spitch));
    const uint4 r2 = __ldg(reinterpret_cast<const uint4*>(s0 + 2 * spitch));
    const uint4 r3 = __ldg(reinterpret_cast<const uint4*>(s0 + 3 * spitch));
    a0 = down4(r0.x, r0.y, r1.x, r1.y);
    a1 = down4(r0.z, r0.w, r1.z, r1.w);
    b0 = down4(r2.x, r2.y, r3.x, r3.y);
    b1 = down4(r2.z, r2.w, r3.z, r3.w);
    *reinterpret_cast<uint2*>(o1) = make_uint2(a0, a1);
    *reinterpret_cast<uint2*>(o1 + p1) = make_uint2(b0, b1);
  } else {
    // ragged edge: byte loads, only in-range pixels
    const int n = min(8, w1 - x8);
    uint8_t v[2][8] = {};
    for (int r = 0; r < (two_rows ? 2 : 1); ++r) {
      const uint8_t* q0 = s0 + static_cast<size_t>(2 * r) * spitch;
      const uint8_t* q1 = q0 + spitch;
      for (int j = 0; j < n; ++j) {
        v[r][j] = static_cast<uint8_t>((q0[2 * j] + q0[2 * j + 1] + q1[2 * j] + q1[2 * j + 1] + 2) >> 2);
        o1[static_cast<size_t>(r) * p1 + j] = v[r][j];
      }
    }
    a0 = v[0][0] | v[0][1] << 8 | v[0][2] << 16 | static_cast<uint32_t>(v[0][3]) << 24;
    a1 = v[0][4] | v[0][5] << 8 | v[0][6] << 16 | static_cast<uint32_t>(v[0][7]) << 24;
    b0 = v[1][0] | v[1][1] << 8 | v[1][2] << 16 | static_cast<uint32_t>(v[1][3]) << 24;
    b1 = v[1][4] | v[1][5] << 8 | v[1][6] << 16 | static_cast<uint32_t>(v[1][7]) << 24;
  }
  const int x4 = x8 >> 1;
  if (ty < h2 && x4 < w2) {  // level-(k+1) pixels need both level-k rows and columns
    const uint32_t c = down4(a0, a1, b0, b1);
    uint8_t* o2 = d2 + f * dfs + static_cast<size_t>(ty) * p2 + x4;
    if (x4 + 4 <= w2) {  // pyramid rows are 16-B aligned
      *reinterpret_cast<uint32_t*>(o2) = c;
    } else {
      for (int j = 0; j < 4 && x4 + j < w2; ++j) o2[j] = static_cast<uint8_t>(c >> (8 * j));
    }
  }
}

// ------------------------------------------------------------------- FAST

template <int N, int KIND>
__global__ void __launch_bounds__(256) k_fast_map(const uint8_t* __restrict__ img, int pitch,
                                                  size_t ifs, int w, int h, int eps,
                                                  uint16_t* __restrict__ resp, int rpitch,
                                                  size_t rfs) {
  const int f = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  int s = 0;
  if (x >= 3 && x < w - 3 && y >= 3 && y < h - 3) {
    const uint8_t* p = img + f * ifs + static_cast<size_t>(y) * pitch + x;
    int ring[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) ring[i] = __ldg(p + ring_dy(i) * pitch + ring_dx(i));
    s = fast_score<N, KIND>(__ldg(p), ring, eps);
  }
  resp[f * rfs + static_cast<size_t>(y) * rpitch + x] = static_cast<uint16_t>(s);
}

// --------------------------------------------------- NMS + cell selection

// Comparisons made by spiral_is_local_max (nms.cpp:48-79): ring r = 1..n,
// top edge left->right, right edge top->bottom, bottom edge right->left,
// left edge bottom->top, in-image neighbours only, stop at the first
// suppressor (inclusive). Returns survival.
__device__ __forceinline__ bool spiral_walk(const uint16_t* __restrict__ r, int rpitch, int w,
                                            int h, int x, int y, int s, int radius,
                                            uint32_t* count) {
  uint32_t c = 0;
  auto visit = [&](int nx, int ny) -> bool {
    if (nx < 0 || ny < 0 || nx >= w || ny >= h) return false;
    ++c;
    const int v = r[static_cast<size_t>(ny) * rpitch + nx];
    return v > s || (v == s && (ny < y || (ny == y && nx < x)));
  };
  for (int k = 1; k <= radius; ++k) {
    for (int dx = -k; dx <= k; ++dx)
      if (visit(x + dx, y - k)) { *count = c; return false; }
    for (int dy = -k + 1; dy <= k; ++dy)
      if (visit(x + k, y + dy)) { *count = c; return false; }
    for (int dx = k - 1; dx >= -k; --dx)
      if (visit(x + dx, y + k)) { *count = c; return false; }
    for (int dy = k - 1; dy >= -k + 1; --dy)
      if (visit(x - k, y + dy)) { *count = c; return false; }
  }
  *count = c;
  return true;
}

template <bool STATS>
__global__ void __launch_bounds__(256) k_nms_select(const uint16_t* __restrict__ resp, int rpitch,
                                                    size_t rfs, int w, int h, int level,
                                                    int radius, int cell_w, int cell_h, int cols,
                                                    int cells, unsigned long long* keys,
                                                    unsigned long long* stats) {
  const int f = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const uint16_t* r = resp + f * rfs;
  uint32_t cand = 0, cmp = 0;
  if (x < w && y < h) {
    const int s = r[static_cast<size_t>(y) * rpitch + x];
    if (s > 0) {
      cand = 1;
      bool keep;
      if (STATS) {
        keep = spiral_walk(r, rpitch, w, h, x, y, s, radius, &cmp);
      } else {
        keep = true;
        const int y0 = max(y - radius, 0), y1 = min(y + radius, h - 1);
        const int x0 = max(x - radius, 0), x1 = min(x + radius, w - 1);
        for (int ny = y0; ny <= y1 && keep; ++ny)
          for (int nx = x0; nx <= x1; ++nx) {
            const int v = r[static_cast<size_t>(ny) * rpitch + nx];
            // an equal neighbour earlier in raster order suppresses
            const bool earlier = ny < y || (ny == y && nx < x);
            if (v > s || (v == s && earlier)) { keep = false; break; }
          }
      }
      if (keep) {
        const int X = x << level, Y = y << level;
        atomicMax(keys + static_cast<size_t>(f) * cells + (Y / cell_h) * cols + X / cell_w,
                  pack_key(s, level, X, Y));
      }
    }
  }
  if (STATS) {
    unsigned long long a = cand, b = cmp;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0 && (a | b)) {
      atomicAdd(stats + 2 * f, a);
      atomicAdd(stats + 2 * f + 1, b);
    }
  }
}

// ------------------------------------------------------------ compaction

// One block per frame: the non-empty cell keys, in row-major order, become
// flk_feature records (ballot + popc within a warp, a scan across warps).
// Keys are zeroed behind the read so the next run starts clean.
__global__ void __launch_bounds__(256) k_compact(unsigned long long* __restrict__ keys, int cols,
                                                 int cells, flk_feature* __restrict__ feats,
                                                 int* __restrict__ counts) {
  __shared__ int warp_base[33];
  const int f = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long* k = keys + static_cast<size_t>(f) * cells;
  flk_feature* out = feats + static_cast<size_t>(f) * cells;
  int base = 0;
  for (int c0 = 0; c0 < cells; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    unsigned long long key = 0;
    if (i < cells) {
      key = k[i];
      if (key) k[i] = 0;
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, key != 0);
    if (lane == 0) warp_base[warp] = __popc(ballot);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int j = 0; j < nw; ++j) {
        const int t = warp_base[j];
        warp_base[j] = acc;
        acc += t;
      }
      warp_base[32] = acc;
    }
    __syncthreads();
    if (key) {
      const int slot = base + warp_base[warp] + __popc(ballot & ((1u << lane) - 1u));
      // three 8-byte stores per record (the list may be mapped host memory)
      const flk_feature ft = unpack_key(key, i % cols, i / cols);
      uint2* o = reinterpret_cast<uint2*>(out + slot);
      o[0] = make_uint2(static_cast<uint32_t>(ft.x), static_cast<uint32_t>(ft.y));
      o[1] = make_uint2(__float_as_uint(ft.score), static_cast<uint32_t>(ft.level));
      o[2] = make_uint2(static_cast<uint32_t>(ft.cell_x), static_cast<uint32_t>(ft.cell_y));
    }
    base += warp_base[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[f] = base;
}

}  // namespace flkb
