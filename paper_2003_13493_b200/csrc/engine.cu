// Host orchestration of the sm_100a detector kernels: geometry, device
// buffers, launch plan, stage timing, conformance and synthetic frames.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "conformance.cuh"
#include "engine.hpp"
#include "fused_dispatch.hpp"
#include "kernels_fused.cuh"
#include "kernels_v1.cuh"

namespace flkb {

namespace {

std::atomic<uint64_t> g_launches{0};

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <typename T>
T* dalloc(size_t n, const char* what) {
  void* p = nullptr;
  check_cuda(cudaMalloc(&p, n * sizeof(T) + 16), what);
  return static_cast<T*>(p);
}

using FastFn = void (*)(const uint8_t*, int, size_t, int, int, int, uint16_t*, int, size_t);

template <int N>
FastFn fast_for_kind(int kind) {
  switch (kind) {
    case kSadB: return k_fast_map<N, kSadB>;
    case kSadA: return k_fast_map<N, kSadA>;
    default: return k_fast_map<N, kMt>;
  }
}

FastFn fast_kernel(int n, int kind) {
  switch (n) {
    case 9: return fast_for_kind<9>(kind);
    case 10: return fast_for_kind<10>(kind);
    case 11: return fast_for_kind<11>(kind);
    case 12: return fast_for_kind<12>(kind);
    case 13: return fast_for_kind<13>(kind);
    case 14: return fast_for_kind<14>(kind);
    case 15: return fast_for_kind<15>(kind);
    default: return fast_for_kind<16>(kind);
  }
}

}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

uint64_t launch_count() { return g_launches.load(); }
void count_launches(int n) { g_launches += static_cast<uint64_t>(n); }

DeviceGuard::DeviceGuard(int device) {
  check_cuda(cudaGetDevice(&prev_), "cudaGetDevice");
  if (prev_ != device) check_cuda(cudaSetDevice(device), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur != prev_ && prev_ >= 0) cudaSetDevice(prev_);
}

bool LaunchPlan::set(const std::string& key, int value) {
  if (key == "band_rows") band_rows = value < 0 ? 0 : value;
  else if (key == "tiles") tiles = value < 0 ? 0 : value;
  else if (key == "fuse_pyramid") fuse_pyramid = value < 0 ? -1 : (value != 0);
  else if (key == "pyramid_chunk") pyramid_chunk = value < 0 ? 0 : value;
  else if (key == "pdl") pdl = value != 0;
  else if (key == "list_cap") list_cap = value <= 0 ? 0 : std::max(256, value);
  else if (key == "debug_geom") debug_geom = value != 0;
  else if (key == "staged") staged = value != 0;
  else if (key == "tensor_tma") tensor_tma = value != 0;
  else if (key == "batch_copies") batch_copies = value != 0;
  else return false;
  return true;
}

DetectParams DetectParams::from(const Config& c) {
  DetectParams p;
  p.epsilon = c.epsilon;
  p.arc_length = c.arc_length;
  p.score = static_cast<int>(c.score);
  p.levels = c.num_levels;
  p.radius = c.nms_radius;
  p.cell_w = c.cell_width();
  p.cell_h = c.cell_height();
  return p;
}

Geometry Geometry::make(const DetectParams& p, int width, int height) {
  if (p.levels < 1 || p.levels > kMaxLevels)
    throw InvalidArgument("pyramid needs between 1 and 16 levels");
  if (width < 1 || height < 1) throw InvalidArgument("image dimensions must be positive");
  if ((std::min(width, height) >> (p.levels - 1)) < 8)
    throw InvalidArgument("image " + std::to_string(width) + "x" + std::to_string(height) +
                          " too small for " + std::to_string(p.levels) + " pyramid levels");
  if (width >= (1 << kCoordBits) || height >= (1 << kCoordBits))
    throw InvalidArgument("frames are limited to 262143 pixels per side");
  Geometry g;
  g.width = width;
  g.height = height;
  g.levels = p.levels;
  int w = width, h = height;
  size_t off = 0;
  for (int k = 0; k < p.levels; ++k) {
    g.lw[k] = w;
    g.lh[k] = h;
    g.lpitch[k] = static_cast<int>(round_up(static_cast<size_t>(w), 16));
    if (k > 0) {
      g.loff[k] = off;
      off += static_cast<size_t>(g.lpitch[k]) * h;
    }
    w /= 2;
    h /= 2;
  }
  g.pyr_frame_bytes = round_up(off, 256);
  g.cols = (width + p.cell_w - 1) / p.cell_w;
  g.rows = (height + p.cell_h - 1) / p.cell_h;
  g.cells = g.cols * g.rows;
  return g;
}

namespace {

// Multiply-high constants of the per-level cell maps (Level::cmx ...):
// cx = hi(x * m) + c must equal (x << k) / cell for every coordinate the
// suppression can produce (3 <= x < w - 3); m = ceil(2^(32+k) / cell), or
// m = 2^32 - 1, c = 1 where a cell is one level-k pixel. Verified
// exhaustively; false (-> global-key path) if any level misses.
bool cell_map(uint32_t& m, uint32_t& c, int k, int cell, int extent) {
  if (cell < (1 << k)) return false;
  if (cell == (1 << k)) {
    m = 0xFFFFFFFFu, c = 1;
  } else {
    const uint64_t num = uint64_t{1} << (32 + k);  // k < kMaxLevels: fits
    const uint64_t q = (num + static_cast<uint64_t>(cell) - 1) / static_cast<uint64_t>(cell);
    if (q >> 32) return false;
    m = static_cast<uint32_t>(q), c = 0;
  }
  for (int x = 3; x < extent - 3; ++x) {
    const uint32_t got = static_cast<uint32_t>((static_cast<uint64_t>(x) * m) >> 32) + c;
    if (got != static_cast<uint32_t>((static_cast<int64_t>(x) << k) / cell)) return false;
  }
  return true;
}

}  // namespace

DeviceBatch::DeviceBatch(const DetectParams& p, int device, int width, int height, int capacity)
    : p_(p), g_(Geometry::make(p, width, height)), device_(device), capacity_(capacity) {
  if (capacity < 1) throw InvalidArgument("batch capacity must be positive");
  DeviceGuard guard(device_);
  size_t resp = 0;
  for (int k = 0; k < g_.levels; ++k) resp += static_cast<size_t>(g_.lpitch[k]) * g_.lh[k];
  resp_frame_elems_ = round_up(resp, 128);
  const size_t cap = static_cast<size_t>(capacity_);
  if (g_.pyr_frame_bytes) d_pyr_ = dalloc<uint8_t>(g_.pyr_frame_bytes * cap, "pyramid");
  d_resp_ = dalloc<uint16_t>(resp_frame_elems_ * cap, "responses");
  d_keys_ = dalloc<unsigned long long>(static_cast<size_t>(g_.cells) * cap, "cell keys");
  d_feats_ = dalloc<flk_feature>(static_cast<size_t>(g_.cells) * cap, "features");
  d_counts_ = dalloc<int>(cap, "counts");
  d_stats_ = dalloc<uint64_t>(2 * cap, "stats");
  d_phase_ = dalloc<unsigned long long>(2, "phase cycles");
  check_cuda(cudaMemset(d_keys_, 0, sizeof(unsigned long long) * g_.cells * cap), "memset keys");
  // the staged score maps' pitch padding is never written: zeroed once so a
  // whole-map download reads defined bytes
  check_cuda(cudaMemset(d_resp_, 0, sizeof(uint16_t) * resp_frame_elems_ * cap), "memset responses");
  // feature slots past a frame's count are never written; the batch download
  // copies whole frame slots
  check_cuda(cudaMemset(d_feats_, 0, sizeof(flk_feature) * g_.cells * cap), "memset features");
  check_cuda(cudaMemset(d_counts_, 0, sizeof(int) * cap), "memset counts");
  check_cuda(cudaMemset(d_stats_, 0, sizeof(uint64_t) * 2 * cap), "memset stats");
  cell_ok_ = true;
  for (int k = 0; k < g_.levels && cell_ok_; ++k)
    cell_ok_ = cell_map(cmap_[k][0], cmap_[k][1], k, p_.cell_w, g_.lw[k]) &&
               cell_map(cmap_[k][2], cmap_[k][3], k, p_.cell_h, g_.lh[k]);
}

DeviceBatch::~DeviceBatch() {
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  cudaFree(d_pyr_);
  cudaFree(d_resp_);
  cudaFree(d_keys_);
  cudaFree(d_feats_);
  cudaFree(d_counts_);
  cudaFree(d_stats_);
  cudaFree(d_phase_);
  for (cudaEvent_t e : evs_) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  cudaFree(d_naive_);
  cudaFree(d_conf_);
  if (cur >= 0) cudaSetDevice(cur);
}

int DeviceBatch::kernels_per_run() const { return last_launches_ ? last_launches_ : g_.levels + 1; }

namespace {

// cuTensorMapEncodeTiled from the driver through the runtime's entry-point
// query (the library links no libcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// The fused kernel's staging map of one level: u8 (x, y, frame) over
// `frames` frames, box = (stage pitch, stage rows, 1). False if the shape
// does not fit a TMA box or the encoder is unavailable (row copies then).
bool encode_stage_map(fused::Level& L, int frames, int box_w, int box_h) {
  auto enc = tensor_map_encoder();
  if (!enc || !L.tma || box_w > 256 || box_h > 256 || box_w % 16) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(L.w), static_cast<cuuint64_t>(L.h),
                              static_cast<cuuint64_t>(frames)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(L.pitch), static_cast<cuuint64_t>(L.fstride)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(&L.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(L.img), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The launch's per-CTA geometry table (fused::Params::geo): level, rows,
// columns and in-CTA cell range of each CTA, packed in 16-bit fields; empty
// (the kernel computes its own) when the launch has more CTAs than the table
// holds or a field does not fit.
void fill_geometry(fused::Params& P, int kb, int ke, int ctas) {
  P.geo_n = 0;
  if (ctas > fused::kGeoMax) return;
  int i = 0;
  for (int k = kb; k < ke; ++k) {
    const fused::Level& L = P.lv[k];
    for (int local = 0; local < L.bands * L.tiles_x; ++local, ++i) {
      const int band = local / L.tiles_x, tile = local % L.tiles_x;
      const int y0 = band * P.R, y1 = std::min(y0 + P.R, L.h);
      const int x_lo = tile * L.tile_w, x_hi = std::min(x_lo + L.tile_w, L.w);
      const int cr0 = (y0 << k) / P.cell_h;
      const int nrows = (y1 > y0 ? ((y1 - 1) << k) / P.cell_h : cr0) - cr0 + 1;
      const int cc0 = (x_lo << k) / P.cell_w;
      const int ccols = (x_hi > x_lo ? ((x_hi - 1) << k) / P.cell_w : cc0) - cc0 + 1;
      const int v[8] = {y0, y1, x_lo, x_hi, cr0, cc0, ccols, nrows};
      for (int x : v)
        if (x < 0 || x > 0xFFFF) return;
      if (k > 15 || nrows > 4095) return;
      P.geo[i] = make_uint4(static_cast<uint32_t>(k) | static_cast<uint32_t>(nrows) << 4 |
                                static_cast<uint32_t>(y0) << 16,
                            static_cast<uint32_t>(y1) | static_cast<uint32_t>(x_lo) << 16,
                            static_cast<uint32_t>(x_hi) | static_cast<uint32_t>(cr0) << 16,
                            static_cast<uint32_t>(cc0) | static_cast<uint32_t>(ccols) << 16);
    }
  }
  P.geo_n = ctas;
}

// kMinBlocks CTAs per SM (1 KB of each CTA's share is reserved by the driver)
constexpr int kFusedSmemTarget = (228 * 1024) / fused::kMinBlocks - 1024;
constexpr int kFusedSmemMax = 227 * 1024;

// Shared-memory geometry of the fused kernel for column tiles of at most
// `tile_w` pixels (every level uses the same layout).
fused::Params fused_geometry(const DetectParams& p, const Geometry& g, int R, int tiles0) {
  fused::Params P{};
  P.levels = g.levels;
  P.eps = p.epsilon;
  P.radius = p.radius;
  P.R = R;
  P.cell_w = p.cell_w;
  P.cell_h = p.cell_h;
  P.div_cw = fused::FastDiv::make(static_cast<uint32_t>(p.cell_w));
  P.div_ch = fused::FastDiv::make(static_cast<uint32_t>(p.cell_h));
  P.cols = g.cols;
  P.cells = g.cells;
  const int n = p.radius;
  int tw_max = 1, slots = 0, cta = 0;
  for (int k = 0; k < g.levels; ++k) {
    fused::Level& L = P.lv[k];
    L.w = g.lw[k];
    L.h = g.lh[k];
    // every level uses level 0's tile width; u16 corner-list entries are
    // score-tile indices ((R + 2 radius) rows <= 64 of tiles up to 928 px)
    const int tw0 = std::min((g.lw[0] + tiles0 - 1) / tiles0, 928);
    L.tiles_x = (L.w + tw0 - 1) / tw0;
    L.tile_w = (L.w + L.tiles_x - 1) / L.tiles_x;
    // level-0 tiles start on 16-px boundaries (the fused pyramid's blocks)
    if (k == 0 && L.tiles_x > 1) L.tile_w = (L.tile_w + 15) & ~15;
    L.tiles_x = (L.w + L.tile_w - 1) / L.tile_w;
    L.bands = (L.h + R - 1) / R;
    L.cta0 = cta;
    cta += L.bands * L.tiles_x;
    tw_max = std::max(tw_max, L.tile_w);
    L.nw = 1;
    for (int t = 0; t < L.tiles_x; ++t) {  // the kernel's per-tile word count, maximised
      const int x_lo = t * L.tile_w, x_hi = std::min(x_lo + L.tile_w, L.w);
      const int bx0 = (x_lo - n - 3) & ~15;
      L.nw = std::max(L.nw, (x_hi + n - bx0 - 3 + fused::kOwn - 1) / fused::kOwn);
    }
    L.div_nw = fused::FastDiv::make(static_cast<uint32_t>(L.nw));
    L.div_tiles = fused::FastDiv::make(static_cast<uint32_t>(L.tiles_x));
    // in-CTA keys: the cell rows of R level-k rows x the cell columns of one
    // tile's own columns
    slots = std::max(slots, ((R << k) / p.cell_h + 2) *
                                std::min(g.cols, ((L.tile_w << k) / p.cell_w + 2)));
  }
  P.nw_max = 1;
  for (int k = 0; k < g.levels; ++k) P.nw_max = std::max(P.nw_max, P.lv[k].nw);
  P.sw = static_cast<int>(round_up(
      static_cast<size_t>(std::max(fused::kOwn * (P.nw_max - 1) + 36, tw_max + 2 * n + 22)), 16));
  P.rp = static_cast<int>(round_up(static_cast<size_t>(tw_max + 4 * n), 8));
  // the radius-1 instance has compile-time pitches; layouts that fit are padded to them
  if (n == 1 && P.sw <= fused::kSw1 && P.rp <= fused::kRp1) P.sw = fused::kSw1, P.rp = fused::kRp1;
  P.rp_magic = 0xFFFFFFFFu / static_cast<uint32_t>(P.rp) + 1u;  // ceil(2^32 / rp)
  // 32-bit in-CTA keys (score << 16 | 0xFFFF - the corner's u16 tile index),
  // one shared slot per cell the CTA touches
  P.key_slots = slots <= 4096 ? slots : 0;
  for (int i = 0; i < 32; ++i) P.pow2[i] = 1u << i;
  for (int b = 0; b < 8; ++b) P.emask[b] = ((p.epsilon >> b) & 1) ? 0xFFFFFFFFu : 0u;
  P.neg16eps = 0u - 16u * static_cast<uint32_t>(p.epsilon);
  P.list_cap = p.plan.list_cap;
  return P;
}

}  // namespace

int DeviceBatch::enqueue_pyramid(const uint8_t* frames, size_t fstride, int pitch, int count,
                                 cudaStream_t s, int first, int k0) {
  uint8_t* pyr = d_pyr_ ? d_pyr_ + static_cast<size_t>(first) * g_.pyr_frame_bytes : nullptr;
  int launched = 0;
  for (int k = k0; k < g_.levels;) {
    const uint8_t* src = k == 1 ? frames : pyr + g_.loff[k - 1];
    const int sp = k == 1 ? pitch : g_.lpitch[k - 1];
    const size_t sfs = k == 1 ? fstride : g_.pyr_frame_bytes;
    const int vec_ok = (reinterpret_cast<uintptr_t>(src) % 16 == 0) && sp % 16 == 0 && sfs % 16 == 0;
    if (k + 1 < g_.levels) {
      dim3 block(32, 8), grid((g_.lw[k] + 255) / 256, (g_.lh[k] + 15) / 16, count);
      k_pyramid_down2<<<grid, block, 0, s>>>(src, sp, sfs, pyr + g_.loff[k], g_.lpitch[k],
                                             pyr + g_.loff[k + 1], g_.lpitch[k + 1],
                                             g_.pyr_frame_bytes, g_.lw[k], g_.lh[k], g_.lw[k + 1],
                                             g_.lh[k + 1], vec_ok);
      k += 2;
    } else {
      dim3 block(32, 8), grid((g_.lw[k] + 255) / 256, (g_.lh[k] + 7) / 8, count);
      k_pyramid_down<<<grid, block, 0, s>>>(src, sp, sfs, pyr + g_.loff[k], g_.lpitch[k],
                                            g_.pyr_frame_bytes, g_.lw[k], g_.lh[k], vec_ok);
      k += 1;
    }
    ++launched;
  }
  return launched;
}

void DeviceBatch::build_pyramid(const uint8_t* frames, size_t fstride, int pitch, int count,
                                cudaStream_t s, int first) {
  if (count < 1 || first < 0 || first + count > capacity_)
    throw InvalidArgument("batch count outside the batch capacity");
  DeviceGuard guard(device_);
  const int n = enqueue_pyramid(frames, fstride, pitch, count, s, first);
  check_cuda(cudaGetLastError(), "pyramid launch");
  count_launches(n);
}

void DeviceBatch::run(const uint8_t* frames, size_t fstride, int pitch, int count, bool stats,
                      cudaStream_t s, StageTimes* times, int first, bool pyramid_ready,
                      int* out_counts, flk_feature* out_feats) {
  if (count < 1 || first < 0 || first + count > capacity_)
    throw InvalidArgument("batch count " + std::to_string(count) + " outside [1, " +
                          std::to_string(capacity_) + "]");
  if (pitch < g_.width) throw InvalidArgument("row pitch smaller than the frame width");
  if (count > 65535) throw InvalidArgument("at most 65535 frames per launch");
  DeviceGuard guard(device_);
  int R = fused_R_;
  const int r_min = 8;
  const LaunchPlan& plan = p_.plan;
  const bool forced = plan.band_rows > 0;  // tuning / test override
  // u16 corner-list entries are score-tile indices: R + 2 radius <= 64
  const int r_max = std::max(4, (64 - 2 * p_.radius) & ~3);
  if (forced) R = std::min(r_max, std::max(4, plan.band_rows));
  const bool forced_tiles = plan.tiles > 0;  // tuning / test override
  int tiles0 = forced_tiles ? plan.tiles : 1;
  fused::Params P = fused_geometry(p_, g_, R, tiles0);
  if (!forced && !forced_tiles && fused_tiles0_ > 0) {
    R = fused_R_, tiles0 = fused_tiles0_;
    P = fused_geometry(p_, g_, R, tiles0);
  } else if (!forced && !forced_tiles) {
    // Pick (band rows, column tiles) with the least halo work among the
    // shapes that fit kMinBlocks CTAs per SM: plane words cost ~0.3, mask
    // words ~0.7 per row, plus a fixed per-CTA share (setup, NMS, flush).
    // Radius 1 keeps to column tiles the compile-time-pitch instance takes
    // (at most 192 px), unless no such shape fits.
    double best = 1e300;
    const int t_max = p_.radius == 1 ? std::max(8, g_.lw[0] / 176 + 1) : 8;
    for (int pass = 0; pass < 2 && best == 1e300; ++pass) {
      for (int r = std::min(r_max, 40); r >= 12; r -= 4) {
        for (int t = 1; t <= t_max; ++t) {
          const fused::Params q = fused_geometry(p_, g_, r, t);
          if (fused::smem_layout(q).total > kFusedSmemTarget) continue;
          if (pass == 0 && p_.radius == 1 && q.sw != fused::kSw1) continue;
          const int n = p_.radius;
          double cost = 0;
          for (int k = 0; k < q.levels; ++k)
            cost += double(q.lv[k].bands) * q.lv[k].tiles_x * q.lv[k].nw *
                    (0.3 * (r + 2 * n + 6) + 0.7 * (r + 2 * n) + 4.0);
          if (cost < best) best = cost, R = r, tiles0 = t, P = q;
          break;  // more tiles at the same r only add column halo
        }
      }
    }
    if (best < 1e300) fused_R_ = R, fused_tiles0_ = tiles0;
  }
  while (fused::smem_layout(P).total > kFusedSmemTarget && P.lv[0].tile_w > 64) {
    ++tiles0;
    P = fused_geometry(p_, g_, R, tiles0);
  }
  // Small batches (the single-frame latency path): trade halo work for
  // parallelism until the grid covers the GPU.
  auto ctas_of = [&](const fused::Params& q) {
    int c = 0;
    for (int k = 0; k < q.levels; ++k) c += q.lv[k].bands * q.lv[k].tiles_x;
    return c * count;
  };
  while (!forced && ctas_of(P) < 2 * 148 && R - 4 >= r_min) {
    R -= 4;
    P = fused_geometry(p_, g_, R, tiles0);
  }
  while (!forced && ctas_of(P) < 148 && P.lv[0].tile_w > 128 && tiles0 < 8) {
    ++tiles0;
    P = fused_geometry(p_, g_, R, tiles0);
  }
  if (!cell_ok_) P.key_slots = 0;  // no exact cell maps: global cell keys
  // the corner list takes whatever the kMinBlocks-per-SM budget leaves (dense
  // levels otherwise score a band in several rounds)
  if (P.list_cap == 0) {
    const int spare = (kFusedSmemTarget - fused::smem_layout(P).total) / 2 & ~7;
    if (spare > 0) P.list_cap = fused::smem_layout(P).list_entries + spare;
  }
  for (int k = 0; k < g_.levels && cell_ok_; ++k) {
    P.lv[k].cmx = cmap_[k][0];
    P.lv[k].ccx = cmap_[k][1];
    P.lv[k].cmy = cmap_[k][2];
    P.lv[k].ccy = cmap_[k][3];
  }
  if (dump_scores_) {  // the staged maps' layout: level k at pitch lpitch[k], levels back to back
    size_t off = 0;
    for (int k = 0; k < g_.levels; ++k) {
      P.lv[k].dbg_off = off;
      P.lv[k].dbg_pitch = g_.lpitch[k];
      off += static_cast<size_t>(g_.lpitch[k]) * g_.lh[k];
    }
    P.dbg_map = d_resp_ + static_cast<size_t>(first) * resp_frame_elems_;
    P.dbg_fstride = resp_frame_elems_;
  }
  fused::finalize(P);
  const int smem = fused::smem_layout(P).total;
  if (plan.debug_geom)
    std::fprintf(stderr, "flkb: R=%d tiles0=%d smem=%d ctas=%d\n", R, tiles0, smem, ctas_of(P));
  // pathological radius (or the staged plan asked for): the staged kernels
  // (corner-list entries are u16 score-tile indices: (R + 2 radius) rows x rp)
  if (smem > kFusedSmemMax || R + 2 * p_.radius > 64 || (R + 2 * p_.radius) * P.rp > 65536 ||
      plan.staged) {
    run_staged(frames, fstride, pitch, count, stats, s, times, first);
    if (out_counts)
      check_cuda(cudaMemcpyAsync(out_counts, d_counts_ + first, sizeof(int) * count,
                                 cudaMemcpyDefault, s), "counts out");
    if (out_feats)
      check_cuda(cudaMemcpyAsync(out_feats, d_feats_ + static_cast<size_t>(first) * g_.cells,
                                 sizeof(flk_feature) * g_.cells * count, cudaMemcpyDefault, s),
                 "features out");
    return;
  }
  const bool fixed_pitch = p_.radius == 1 && P.sw == fused::kSw1 && P.rp == fused::kRp1;
  const fused::KernelFn kern = fused::kernel_for(p_.arc_length, p_.score, fixed_pitch ? 1 : 0, stats);
  if (reinterpret_cast<const void*>(kern) != fused_kern_ || static_cast<size_t>(smem) > fused_smem_) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "fused smem attribute");
    if (reinterpret_cast<const void*>(kern) != fused_kern_) fused_smem_ = 0;
    fused_kern_ = reinterpret_cast<const void*>(kern);
    fused_smem_ = std::max(fused_smem_, static_cast<size_t>(smem));
  }
  uint8_t* pyr = d_pyr_ ? d_pyr_ + static_cast<size_t>(first) * g_.pyr_frame_bytes : nullptr;
  unsigned long long* keys = d_keys_ + static_cast<size_t>(first) * g_.cells;
  flk_feature* feats = out_feats ? out_feats : d_feats_ + static_cast<size_t>(first) * g_.cells;
  int* counts = out_counts ? out_counts : d_counts_ + first;
  unsigned long long* st =
      reinterpret_cast<unsigned long long*>(d_stats_ + 2 * static_cast<size_t>(first));

  // Pyramid levels 1 (and 2) come out of the level-0 CTAs of the fused kernel
  // (one HBM pass over level 0 instead of two) when the band and tile shape
  // keep their 16x4 blocks aligned; the remaining levels are detected by a
  // second launch once the pyramid exists. Small batches keep the one-launch
  // plan: there a level-0-only launch would not fill the GPU.
  const int ctas0 = P.lv[0].bands * P.lv[0].tiles_x;
  const bool aligned =
      g_.levels >= 2 && R % 4 == 0 && (P.lv[0].tiles_x == 1 || P.lv[0].tile_w % 16 == 0);
  bool want = static_cast<long>(ctas0) * count >= 4L * 148 * fused::kMinBlocks;
  if (plan.fuse_pyramid >= 0) want = plan.fuse_pyramid != 0;  // tests / tuning
  const int fuse_pyr = aligned && want && !pyramid_ready ? std::min(2, g_.levels - 1) : 0;

  cudaEvent_t ev[5] = {};
  if (times) {
    for (auto& e : ev) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    check_cuda(cudaEventRecord(ev[0], s), "cudaEventRecord");
  }
  if (stats) check_cuda(cudaMemsetAsync(st, 0, sizeof(uint64_t) * 2 * count, s), "memset stats");
  // a timed stats run splits the fused launches' time into the response and
  // the suppression phases by the kernel's own cycle counts
  const bool split = stats && times;
  if (split) {
    check_cuda(cudaMemsetAsync(d_phase_, 0, 2 * sizeof(unsigned long long), s), "memset phases");
    P.phase_cycles = d_phase_;
  }
  int launched = 0;
  // frame pointers of the frames [c0, c0 + n) of this call
  auto bind = [&](int c0, int nf) {
    for (int k = 0; k < g_.levels; ++k) {
      fused::Level& L = P.lv[k];
      L.img = k == 0 ? frames + static_cast<size_t>(c0) * fstride
                     : pyr + static_cast<size_t>(c0) * g_.pyr_frame_bytes + g_.loff[k];
      L.pitch = k == 0 ? pitch : g_.lpitch[k];
      L.fstride = k == 0 ? fstride : g_.pyr_frame_bytes;
      L.tma = (reinterpret_cast<uintptr_t>(L.img) % 16 == 0) && L.pitch % 16 == 0 &&
              L.fstride % 16 == 0;
      if (k > 0 && k < 3) P.pyr_img[k] = const_cast<uint8_t*>(L.img);
      L.tmap_ok = plan.tensor_tma && encode_stage_map(L, nf, P.sw, P.R + 2 * p_.radius + 6);
    }
    P.keys = keys + static_cast<size_t>(c0) * g_.cells;
    if (dump_scores_)
      P.dbg_map = d_resp_ + static_cast<size_t>(first + c0) * resp_frame_elems_;
    P.stats = stats ? st + 2 * static_cast<size_t>(c0) : nullptr;
  };
  // detection of levels [kb, ke) of n frames in one launch
  auto detect = [&](int kb, int ke, int pyr_levels, int n, cudaStream_t ls) {
    P.k_begin = kb;
    P.k_end = ke;
    P.pyr_levels = pyr_levels;
    int ctas = 0;
    for (int k = kb; k < ke; ++k) {
      P.lv[k].cta0 = ctas;
      ctas += P.lv[k].bands * P.lv[k].tiles_x;
    }
    fill_geometry(P, kb, ke, ctas);
    if (P.pdl_wait) {  // overlap the pyramid kernel (and this launch's latency)
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(ctas, n);
      lc.blockDim = dim3(fused::kThreads);
      lc.dynamicSmemBytes = smem;
      lc.stream = ls;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      check_cuda(cudaLaunchKernelEx(&lc, kern, P), "fused launch (programmatic)");
    } else {
      kern<<<dim3(ctas, n), fused::kThreads, smem, ls>>>(P);
    }
    ++launched;
  };
  // Two-launch plan in chunks of frames whose pyramid levels 1-2 fit in L2:
  // the level 1-2 launch of a chunk reads what the level-0 launch just wrote
  // from L2 instead of HBM.
  // (equal chunks of at most 32 MiB of levels 1-2: a quarter of the L2)
  int chunk = count;
  if (fuse_pyr) {
    size_t b12 = 0;
    for (int k = 1; k <= fuse_pyr; ++k) b12 += static_cast<size_t>(g_.lpitch[k]) * g_.lh[k];
    const size_t nchunks = (static_cast<size_t>(count) * b12 + (32u << 20) - 1) / (32u << 20);
    chunk = static_cast<int>((count + nchunks - 1) / std::max<size_t>(nchunks, 1));
  }
  if (plan.pyramid_chunk > 0) chunk = plan.pyramid_chunk;
  if (fuse_pyr) {
    if (times) check_cuda(cudaEventRecord(ev[1], s), "cudaEventRecord");
    if (times) check_cuda(cudaEventRecord(ev[2], s), "cudaEventRecord");
    // chunk i's level 1-2 launch runs on a side stream, overlapping chunk
    // i+1's level-0 launch (their tails fill each other's idle SMs)
    const bool overlap = chunk < count;
    cudaStream_t s1 = s;
    if (overlap) {
      if (!side_) check_cuda(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "side stream");
      const size_t need = 2 * static_cast<size_t>((count + chunk - 1) / chunk) + 1;
      while (evs_.size() < need) {
        cudaEvent_t e;
        check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        evs_.push_back(e);
      }
      s1 = side_;
      check_cuda(cudaEventRecord(evs_[0], s), "fork");
      check_cuda(cudaStreamWaitEvent(side_, evs_[0], 0), "fork wait");
    }
    int ei = 1;
    for (int c0 = 0; c0 < count; c0 += chunk) {
      const int n = std::min(chunk, count - c0);
      bind(c0, n);
      detect(0, 1, fuse_pyr, n, s);
      launched += enqueue_pyramid(frames + static_cast<size_t>(c0) * fstride, fstride, pitch, n, s,
                                  first + c0, fuse_pyr + 1);
      if (overlap) {
        check_cuda(cudaEventRecord(evs_[ei], s), "chunk level 0 done");
        check_cuda(cudaStreamWaitEvent(side_, evs_[ei], 0), "chunk wait");
        ++ei;
      }
      detect(1, g_.levels, 0, n, s1);
    }
    if (overlap) {
      check_cuda(cudaEventRecord(evs_[ei], side_), "join");
      check_cuda(cudaStreamWaitEvent(s, evs_[ei], 0), "join wait");
    }
  } else {
    bind(0, count);
    int pyr_launches = 0;
    if (!pyramid_ready) pyr_launches = enqueue_pyramid(frames, fstride, pitch, count, s, first);
    launched += pyr_launches;
    if (times) check_cuda(cudaEventRecord(ev[1], s), "cudaEventRecord");
    if (times) check_cuda(cudaEventRecord(ev[2], s), "cudaEventRecord");
    P.pdl_wait = plan.pdl && pyr_launches > 0 && !times;
    detect(0, g_.levels, 0, count, s);
    P.pdl_wait = 0;
  }
  if (times) check_cuda(cudaEventRecord(ev[3], s), "cudaEventRecord");
  k_compact<<<count, 256, 0, s>>>(keys, g_.cols, g_.cells, feats, counts);
  ++launched;
  check_cuda(cudaGetLastError(), "kernel launch");
  count_launches(launched);
  last_launches_ = launched;
  if (times) {
    check_cuda(cudaEventRecord(ev[4], s), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(ev[4]), "cudaEventSynchronize");
    float a = 0, b = 0, c = 0, d = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    cudaEventElapsedTime(&d, ev[3], ev[4]);
    // pyramid_us: the downsampling launches; the fused launches compute
    // responses and suppression together (and, in the two-launch plan,
    // pyramid levels 1-2): with stats their time is split by the kernel's
    // phase cycles into crf_us (staging .. scoring) and nms_us (suppression,
    // cell selection) plus the compaction, as frontend.cpp:42-53 times the
    // two stages; without stats crf_us is the whole fused time and nms_us the
    // compaction.
    const double fused = (fuse_pyr ? a + c : c) * 1e3;
    times->pyramid_us = (fuse_pyr ? b : a) * 1e3;
    times->crf_us = fused;
    times->nms_us = d * 1e3;
    if (split) {
      unsigned long long cyc[2] = {0, 0};
      check_cuda(cudaMemcpy(cyc, d_phase_, sizeof(cyc), cudaMemcpyDeviceToHost), "phase cycles");
      const double tot = static_cast<double>(cyc[0]) + static_cast<double>(cyc[1]);
      if (tot > 0) {
        times->crf_us = fused * static_cast<double>(cyc[0]) / tot;
        times->nms_us += fused * static_cast<double>(cyc[1]) / tot;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void DeviceBatch::run_staged(const uint8_t* frames, size_t fstride, int pitch, int count,
                             bool stats, cudaStream_t s, StageTimes* times, int first) {
  if (count < 1 || first < 0 || first + count > capacity_)
    throw InvalidArgument("batch count " + std::to_string(count) + " outside [1, " +
                          std::to_string(capacity_) + "]");
  if (pitch < g_.width) throw InvalidArgument("row pitch smaller than the frame width");
  DeviceGuard guard(device_);
  cudaEvent_t ev[4] = {};
  if (times) {
    for (auto& e : ev) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    check_cuda(cudaEventRecord(ev[0], s), "cudaEventRecord");
  }
  // outputs of frame f land in slot first + f
  uint8_t* pyr = d_pyr_ ? d_pyr_ + static_cast<size_t>(first) * g_.pyr_frame_bytes : nullptr;
  uint16_t* respb = d_resp_ + static_cast<size_t>(first) * resp_frame_elems_;
  unsigned long long* keys = d_keys_ + static_cast<size_t>(first) * g_.cells;
  flk_feature* feats = d_feats_ + static_cast<size_t>(first) * g_.cells;
  int* counts = d_counts_ + first;
  unsigned long long* st = reinterpret_cast<unsigned long long*>(d_stats_ + 2 * static_cast<size_t>(first));
  if (stats) check_cuda(cudaMemsetAsync(st, 0, sizeof(uint64_t) * 2 * count, s), "memset stats");

  // level k's image: base pointer, pitch, frame stride
  auto level_ptr = [&](int k) -> const uint8_t* { return k == 0 ? frames : pyr + g_.loff[k]; };
  auto level_pitch = [&](int k) { return k == 0 ? pitch : g_.lpitch[k]; };
  auto level_fs = [&](int k) { return k == 0 ? fstride : g_.pyr_frame_bytes; };

  int launched = 0;
  for (int k = 1; k < g_.levels; ++k) {
    const int wd = g_.lw[k], hd = g_.lh[k];
    const uint8_t* src = level_ptr(k - 1);
    const int vec_ok = (reinterpret_cast<uintptr_t>(src) % 16 == 0) && level_pitch(k - 1) % 16 == 0 &&
                       level_fs(k - 1) % 16 == 0;
    dim3 block(32, 8), grid((wd + 255) / 256, (hd + 7) / 8, count);
    k_pyramid_down<<<grid, block, 0, s>>>(src, level_pitch(k - 1), level_fs(k - 1),
                                          pyr + g_.loff[k], g_.lpitch[k], g_.pyr_frame_bytes,
                                          wd, hd, vec_ok);
    ++launched;
  }
  if (times) check_cuda(cudaEventRecord(ev[1], s), "cudaEventRecord");

  size_t roff = 0;
  size_t roffs[kMaxLevels];
  const FastFn fast = fast_kernel(p_.arc_length, p_.score);
  for (int k = 0; k < g_.levels; ++k) {
    roffs[k] = roff;
    dim3 block(64, 4), grid((g_.lw[k] + 63) / 64, (g_.lh[k] + 3) / 4, count);
    fast<<<grid, block, 0, s>>>(level_ptr(k), level_pitch(k), level_fs(k), g_.lw[k], g_.lh[k],
                                p_.epsilon, respb + roff, g_.lpitch[k], resp_frame_elems_);
    roff += static_cast<size_t>(g_.lpitch[k]) * g_.lh[k];
    ++launched;
  }
  if (times) check_cuda(cudaEventRecord(ev[2], s), "cudaEventRecord");

  for (int k = 0; k < g_.levels; ++k) {
    dim3 block(64, 4), grid((g_.lw[k] + 63) / 64, (g_.lh[k] + 3) / 4, count);
    if (stats)
      k_nms_select<true><<<grid, block, 0, s>>>(respb + roffs[k], g_.lpitch[k], resp_frame_elems_,
                                                g_.lw[k], g_.lh[k], k, p_.radius, p_.cell_w,
                                                p_.cell_h, g_.cols, g_.cells, keys, st);
    else
      k_nms_select<false><<<grid, block, 0, s>>>(respb + roffs[k], g_.lpitch[k], resp_frame_elems_,
                                                 g_.lw[k], g_.lh[k], k, p_.radius, p_.cell_w,
                                                 p_.cell_h, g_.cols, g_.cells, keys, nullptr);
    ++launched;
  }
  k_compact<<<count, 256, 0, s>>>(keys, g_.cols, g_.cells, feats, counts);
  ++launched;
  check_cuda(cudaGetLastError(), "kernel launch");
  count_launches(launched);
  if (times) {
    check_cuda(cudaEventRecord(ev[3], s), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(ev[3]), "cudaEventSynchronize");
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    times->pyramid_us = a * 1e3;
    times->crf_us = b * 1e3;
    times->nms_us = c * 1e3;
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void DeviceBatch::download(int first, int count, int* counts, flk_feature* feats,
                           cudaStream_t s) const {
  if (first < 0 || count < 0 || first + count > capacity_)
    throw InvalidArgument("download range outside the batch");
  DeviceGuard guard(device_);
  if (counts)
    check_cuda(cudaMemcpyAsync(counts, d_counts_ + first, sizeof(int) * count,
                               cudaMemcpyDeviceToHost, s), "download counts");
  if (feats)
    check_cuda(cudaMemcpyAsync(feats, d_feats_ + static_cast<size_t>(first) * g_.cells,
                               sizeof(flk_feature) * g_.cells * count, cudaMemcpyDeviceToHost, s),
               "download features");
}

void DeviceBatch::download_responses(int frame, float* out, cudaStream_t s) const {
  DeviceGuard guard(device_);
  std::vector<uint16_t> tmp(resp_frame_elems_);
  check_cuda(cudaMemcpyAsync(tmp.data(), d_resp_ + static_cast<size_t>(frame) * resp_frame_elems_,
                             sizeof(uint16_t) * resp_frame_elems_, cudaMemcpyDeviceToHost, s),
             "download responses");
  check_cuda(cudaStreamSynchronize(s), "responses sync");
  size_t roff = 0;
  for (int k = 0; k < g_.levels; ++k) {
    for (int y = 0; y < g_.lh[k]; ++y)
      for (int x = 0; x < g_.lw[k]; ++x)
        *out++ = static_cast<float>(tmp[roff + static_cast<size_t>(y) * g_.lpitch[k] + x]);
    roff += static_cast<size_t>(g_.lpitch[k]) * g_.lh[k];
  }
}

flk_conformance DeviceBatch::conformance(const uint8_t* frames, size_t fstride, int pitch,
                                         cudaStream_t s, int first, int count,
                                         flk_conformance* per_frame) {
  if (count < 1 || first < 0 || first + count > capacity_)
    throw InvalidArgument("conformance range outside the batch");
  DeviceGuard guard(device_);
  size_t total = 0;
  for (int k = 0; k < g_.levels; ++k) total += static_cast<size_t>(g_.lw[k]) * g_.lh[k];
  struct Tables {
    int lw[kMaxLevels];
    int lh[kMaxLevels];
    const float* maps[kMaxLevels];
  } t{};
  static_assert(offsetof(Tables, maps) % 8 == 0, "pointer alignment");
  // scratch: one frame's naive maps (reused frame after frame in stream
  // order), the level tables, then 3 tally ints per frame
  if (!d_naive_) d_naive_ = dalloc<float>(total, "conformance maps");
  const size_t need = sizeof(Tables) + 3 * sizeof(int) * static_cast<size_t>(count);
  if (need > conf_bytes_) {
    cudaFree(d_conf_);
    d_conf_ = nullptr;
    d_conf_ = dalloc<int>((need + 3) / 4, "conformance tally");
    conf_bytes_ = need;
  }
  size_t off = 0;
  for (int k = 0; k < g_.levels; ++k) {
    t.lw[k] = g_.lw[k];
    t.lh[k] = g_.lh[k];
    t.maps[k] = d_naive_ + off;
    off += static_cast<size_t>(g_.lw[k]) * g_.lh[k];
  }
  Tables* dt = reinterpret_cast<Tables*>(d_conf_);
  int* tally = reinterpret_cast<int*>(reinterpret_cast<char*>(d_conf_) + sizeof(Tables));
  check_cuda(cudaMemcpyAsync(dt, &t, sizeof(Tables), cudaMemcpyHostToDevice, s), "upload tables");
  check_cuda(cudaMemsetAsync(tally, 0, 3 * sizeof(int) * static_cast<size_t>(count), s), "tally");
  int launched = 0;
  for (int i = 0; i < count; ++i) {
    const int f = first + i;
    int* tf = tally + 3 * i;
    for (int k = 0; k < g_.levels; ++k) {
      const uint8_t* img = k == 0 ? frames + static_cast<size_t>(f) * fstride
                                  : d_pyr_ + static_cast<size_t>(f) * g_.pyr_frame_bytes + g_.loff[k];
      const int ip = k == 0 ? pitch : g_.lpitch[k];
      dim3 block(32, 8), grid((g_.lw[k] + 31) / 32, (g_.lh[k] + 7) / 8);
      k_naive_fast<<<grid, block, 0, s>>>(img, ip, g_.lw[k], g_.lh[k], p_.epsilon, p_.arc_length,
                                          p_.score, const_cast<float*>(t.maps[k]));
      k_naive_survivors<<<grid, block, 0, s>>>(t.maps[k], g_.lw[k], g_.lh[k], p_.radius, tf);
      launched += 2;
    }
    k_conf_features<<<(g_.cells + 127) / 128, 128, 0, s>>>(
        d_feats_ + static_cast<size_t>(f) * g_.cells, d_counts_ + f, dt->maps, dt->lw, dt->lh,
        p_.radius, tf);
    ++launched;
  }
  check_cuda(cudaGetLastError(), "conformance launch");
  count_launches(launched);
  std::vector<int> host(3 * static_cast<size_t>(count));
  check_cuda(cudaMemcpyAsync(host.data(), tally, sizeof(int) * host.size(), cudaMemcpyDeviceToHost,
                             s), "tally");
  check_cuda(cudaStreamSynchronize(s), "conformance sync");
  // tally = naive survivors, matched, false positives (oracle.cpp:240-268)
  flk_conformance sum{0, 0, 0};
  for (int i = 0; i < count; ++i) {
    flk_conformance c;
    c.matched = host[3 * i + 1];
    c.false_positives = host[3 * i + 2];
    c.subset_only = host[3 * i] - host[3 * i + 1];
    if (per_frame) per_frame[i] = c;
    sum.matched += c.matched;
    sum.subset_only += c.subset_only;
    sum.false_positives += c.false_positives;
  }
  return sum;
}

namespace {
__global__ void k_synth(uint8_t* out, int kind, uint64_t first, int w, int h, int pitch,
                        size_t fs) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int f = blockIdx.z;
  if (x >= w || y >= h) return;
  out[f * fs + static_cast<size_t>(y) * pitch + x] = synth_pixel(kind, first + f, x, y, w);
}
}  // namespace

void synth_frames(uint8_t* frames, int kind, uint64_t first, int count, int width, int height,
                  int pitch, size_t fs, cudaStream_t s) {
  if (kind < 0 || kind > 1) throw InvalidArgument("synthetic kind must be 0 (noise) or 1 (texture)");
  dim3 block(64, 4);
  for (int c0 = 0; c0 < count; c0 += 65535) {
    const int n = std::min(65535, count - c0);
    dim3 grid((width + 63) / 64, (height + 3) / 4, n);
    k_synth<<<grid, block, 0, s>>>(frames + c0 * fs, kind, first + c0, width, height, pitch, fs);
    count_launches(1);
  }
  check_cuda(cudaGetLastError(), "synth launch");
}

}  // namespace flkb
