// Detect-track session: GPU pyramid, LK tracking, re-detection and template
// building; host lifecycle in the reference's order (frontend.cpp:65-225).
//
// Bit-exactness of the tracker (fp64): this translation unit is compiled with
// -fmad=false (paper_2003_13493_b200/build.py), so every a*b+c below is a
// rounded product followed by a rounded sum, as the reference's x86-64 build
// (SSE2, no FMA) computes it; every sum that the reference accumulates
// serially (the Hessian entries over the patch, the right-hand side of each
// Gauss-Newton step) is accumulated serially here too, one thread per sum, in
// pixel order. The per-pixel work (bilinear samples, residuals, products) is
// spread over the CTA's threads. std::hypot is glibc's (not correctly rounded:
// ~0.2 % of random pairs differ from the exact rounding), so the device uses
// the same algorithm, glibc_hypot below, rather than CUDA's hypot; it feeds the
// divergence / convergence comparisons (lk.cpp:267, 319).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include <math_constants.h>

#include "session.hpp"

namespace flkb {
namespace lk {

namespace {

__device__ __forceinline__ float sample_bilinear(const uint8_t* __restrict__ img, int pitch, int w,
                                                 int h, double x, double y) {
  // sample_bilinear (image.cpp:67-81); positions are in range by construction
  const int x0 = static_cast<int>(x);
  const int y0 = static_cast<int>(y);
  const int x1 = min(x0 + 1, w - 1);
  const int y1 = min(y0 + 1, h - 1);
  const double fx = x - x0;
  const double fy = y - y0;
  const uint8_t* r0 = img + static_cast<size_t>(y0) * pitch;
  const uint8_t* r1 = img + static_cast<size_t>(y1) * pitch;
  const double top = (1.0 - fx) * r0[x0] + fx * r0[x1];
  const double bot = (1.0 - fx) * r1[x0] + fx * r1[x1];
  return static_cast<float>((1.0 - fy) * top + fy * bot);
}

// glibc 2.35+ __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, the non-FMA kernel an
// x86-64 build without -mfma runs: Borges' correction of sqrt(ax^2 + ay^2)),
// operation for operation, so std::hypot's result is reproduced bit for bit.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

}  // namespace

__device__ double glibc_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) return (isinf(x) || isinf(y)) ? CUDART_INF : x + y;
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return glibc_hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return glibc_hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return glibc_hypot_kernel(ax, ay);
}

namespace {

// det_small (lk.cpp:74-102)
__device__ double det_small(const double* in, int n) {
  double m[16];
  for (int i = 0; i < 16; ++i) m[i] = in[i];
  double det = 1.0;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int row = col + 1; row < n; ++row)
      if (fabs(m[row * n + col]) > fabs(m[pivot * n + col])) pivot = row;
    const double p = m[pivot * n + col];
    if (p == 0.0) return 0.0;
    if (pivot != col) {
      for (int k = 0; k < n; ++k) {
        const double t = m[col * n + k];
        m[col * n + k] = m[pivot * n + k];
        m[pivot * n + k] = t;
      }
      det = -det;
    }
    det *= p;
    for (int row = col + 1; row < n; ++row) {
      const double f = m[row * n + col] / p;
      for (int k = col; k < n; ++k) m[row * n + k] -= f * m[col * n + k];
    }
  }
  return det;
}

// invert_small (lk.cpp:105-143)
__device__ bool invert_small(const double* in, int n, double* out) {
  double m[16], inv[16];
  for (int i = 0; i < 16; ++i) m[i] = in[i], inv[i] = 0.0;
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int row = col + 1; row < n; ++row)
      if (fabs(m[row * n + col]) > fabs(m[pivot * n + col])) pivot = row;
    const double p = m[pivot * n + col];
    if (p == 0.0) return false;
    if (pivot != col) {
      for (int k = 0; k < n; ++k) {
        double t = m[col * n + k];
        m[col * n + k] = m[pivot * n + k];
        m[pivot * n + k] = t;
        t = inv[col * n + k];
        inv[col * n + k] = inv[pivot * n + k];
        inv[pivot * n + k] = t;
      }
    }
    const double scale = 1.0 / p;
    for (int k = 0; k < n; ++k) {
      m[col * n + k] *= scale;
      inv[col * n + k] *= scale;
    }
    for (int row = 0; row < n; ++row) {
      if (row == col) continue;
      const double f = m[row * n + col];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        m[row * n + k] -= f * m[col * n + k];
        inv[row * n + k] -= f * inv[col * n + k];
      }
    }
  }
  for (int i = 0; i < 16; ++i) out[i] = inv[i];
  return true;
}

__host__ __device__ inline bool has_gain(int mode) { return mode == 2 || mode == 3; }
__host__ __device__ inline bool has_offset(int mode) { return mode == 1 || mode == 3; }

// build_template (lk.cpp:147-240) for candidate blockIdx.x at level
// blockIdx.y: one thread per patch pixel, one thread per Hessian entry for
// the serial sums, thread 0 for the 4x4 determinant and inverse. Levels are
// independent; the host accepts a candidate when no level failed and one
// level was usable (the reference stops at the first failing level, which
// gives the same accept/reject decision).
__global__ void __launch_bounds__(256) k_template(Levels lv, const int* __restrict__ cand, int ncand,
                                                  TplLevel* __restrict__ hdr, float* __restrict__ vals,
                                                  double* __restrict__ coef, TrackerParams tp,
                                                  int* __restrict__ tstat) {
  __shared__ double su[kMaxPx][4];
  __shared__ double hess[16];
  const int c = blockIdx.x, k = blockIdx.y, tid = threadIdx.x, L = lv.n;
  const int x0 = cand[2 * c], y0 = cand[2 * c + 1], slot = cand[2 * ncand + c];
  TplLevel* T = hdr + static_cast<size_t>(slot) * L + k;
  const int w = lv.w[k], h = lv.h[k];
  const int patch = k <= 1 ? 16 : 8;
  if (w < patch + 2 || h < patch + 2) {
    if (tid == 0) T->status = tstat[c * L + k] = 3;
    return;
  }
  const int half = patch / 2, npx = patch * patch, dims = tp.dims;
  const double ax = x0 / static_cast<double>(1 << k);
  const double ay = y0 / static_cast<double>(1 << k);
  if (ax - half - 1 < 0.0 || ax + half > w - 1 || ay - half - 1 < 0.0 || ay + half > h - 1) {
    if (tid == 0) T->status = tstat[c * L + k] = 1;
    return;
  }
  const size_t base = (static_cast<size_t>(slot) * L + k) * kMaxPx;
  if (tid < npx) {
    const int oy = -half + tid / patch, ox = -half + tid % patch;
    const double px = ax + ox;
    const double py = ay + oy;
    const uint8_t* img = lv.img[k];
    const int pitch = lv.pitch[k];
    const float value = sample_bilinear(img, pitch, w, h, px, py);
    const float gx = 0.5f * (sample_bilinear(img, pitch, w, h, px + 1, py) -
                             sample_bilinear(img, pitch, w, h, px - 1, py));
    const float gy = 0.5f * (sample_bilinear(img, pitch, w, h, px, py + 1) -
                             sample_bilinear(img, pitch, w, h, px, py - 1));
    vals[base + tid] = value;
    double u[4] = {static_cast<double>(gx), static_cast<double>(gy), 0.0, 0.0};
    int d = 2;
    if (has_gain(tp.mode)) u[d++] = value;
    if (has_offset(tp.mode)) u[d++] = 1.0;
    for (int i = 0; i < 4; ++i) {
      su[tid][i] = u[i];
      coef[(base + tid) * 4 + i] = u[i];
    }
  }
  __syncthreads();
  if (tid < dims * dims) {
    const int r = tid / dims, cc = tid % dims;
    double acc = 0.0;
    for (int i = 0; i < npx; ++i) acc += su[i][r] * su[i][cc];
    hess[tid] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    double hm[16];
    for (int i = 0; i < 16; ++i) hm[i] = i < dims * dims ? hess[i] : 0.0;
    const double det = det_small(hm, dims);
    const double area = static_cast<double>(npx);
    T->level = k;
    T->patch = patch;
    T->dims = dims;
    T->ax = ax;
    T->ay = ay;
    const int st =
        !(det >= tp.min_determinant_factor * area * area) || !invert_small(hm, dims, T->hinv) ? 2 : 0;
    T->status = tstat[c * L + k] = st;
  }
}

// track_feature (lk.cpp:242-350) for track blockIdx.x: coarse to fine over
// the template's levels; per iteration one thread per pixel computes the
// residual and its products with the coefficients, one thread per parameter
// sums them in pixel order, and every thread then applies the identical
// update (deterministic, no broadcast needed).
__global__ void __launch_bounds__(256) k_track(Levels lv, const int* __restrict__ n_tracks,
                                               const TrackIO* __restrict__ io,
                                               TrackIO* __restrict__ io_out,
                                               const TplLevel* __restrict__ hdr,
                                               const float* __restrict__ vals,
                                               const double* __restrict__ coef, TrackerParams tp) {
  __shared__ double prod[4][kMaxPx];
  __shared__ double rhs[4];
  __shared__ double hinv_s[16];
  __shared__ TrackIO rec;
  __shared__ int live;
  const int t = blockIdx.x, tid = threadIdx.x, L = lv.n;
  if (tid == 0) {
    live = *n_tracks;
    if (t < live) rec = io[t];
  }
  __syncthreads();
  if (t >= live) return;  // the frame graph launches one CTA per slot
  const int slot = rec.slot;
  double tx0 = rec.w[0], ty0 = rec.w[1], gain = rec.w[2], offset = rec.w[3];
  int iters = 0, status = 0;
  bool aborted = false, finest_converged = false;
  int finest = -1;
  for (int k = 0; k < L && finest < 0; ++k)
    if (hdr[static_cast<size_t>(slot) * L + k].status == 0) finest = k;
  for (int k = L - 1; k >= 0; --k) {
    const TplLevel& T = hdr[static_cast<size_t>(slot) * L + k];
    if (T.status != 0) continue;
    const uint8_t* img = lv.img[k];
    const int pitch = lv.pitch[k], w = lv.w[k], h = lv.h[k];
    const double scale = static_cast<double>(1 << k);
    double tx = tx0 / scale;
    double ty = ty0 / scale;
    const int patch = T.patch, half = patch / 2, npx = patch * patch, dims = T.dims;
    const double ax = T.ax, ay = T.ay;
    const double max_step = 0.5 * glibc_hypot(static_cast<double>(w), static_cast<double>(h));
    const size_t base = (static_cast<size_t>(slot) * L + k) * kMaxPx;
    // the level's inverse Hessian in shared memory (read by every thread for
    // the identical update each iteration)
    __syncthreads();  // the previous level's last update has read hinv_s
    if (tid < 16) hinv_s[tid] = T.hinv[tid];
    __syncthreads();
    // this thread's template pixel, fixed for the level: kept in registers
    const int oy = -half + tid / patch, ox = -half + tid % patch;
    double tv = 0.0, u[4] = {0.0, 0.0, 0.0, 0.0};
    if (tid < npx) {
      tv = vals[base + tid];
      for (int d = 0; d < dims; ++d) u[d] = coef[(base + tid) * 4 + d];
    }
    bool level_converged = false;
    for (int iter = 0; iter < tp.max_iterations; ++iter) {
      const double bx0 = ax - half + tx;
      const double bx1 = ax + half - 1 + tx;
      const double by0 = ay - half + ty;
      const double by1 = ay + half - 1 + ty;
      if (bx0 < 0.0 || by0 < 0.0 || bx1 > w - 1 || by1 > h - 1) {
        status = 2;  // OUT_OF_BOUNDS
        aborted = true;
        break;
      }
      if (tid < npx) {
        const double sample = sample_bilinear(img, pitch, w, h, ax + ox + tx, ay + oy + ty);
        const double r = sample - (1.0 + gain) * tv - offset;
        for (int d = 0; d < dims; ++d) prod[d][tid] = u[d] * r;
      }
      __syncthreads();
      if (tid < dims) {
        double acc = 0.0;
        for (int i = 0; i < npx; ++i) acc += prod[tid][i];
        rhs[tid] = acc;
      }
      __syncthreads();
      double delta[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = 0; r < dims; ++r) {
        double acc = 0.0;
        for (int c = 0; c < dims; ++c) acc += hinv_s[r * dims + c] * rhs[c];
        delta[r] = acc;
      }
      ++iters;
      tx -= delta[0];
      ty -= delta[1];
      int d = 2;
      if (has_gain(tp.mode)) gain += delta[d++];
      if (has_offset(tp.mode)) offset += delta[d++];
      const double step = glibc_hypot(delta[0], delta[1]);
      if (step > max_step || !(gain > -1.0) || !isfinite(step)) {
        status = 1;  // DIVERGED
        aborted = true;
        break;
      }
      if (step <= tp.convergence_epsilon) {
        level_converged = true;
        break;
      }
    }
    tx0 = tx * scale;
    ty0 = ty * scale;
    if (aborted) break;
    if (k == finest) finest_converged = level_converged;
  }
  if (!aborted && !finest_converged) status = 4;  // MAX_ITERATIONS
  if (tid == 0) {  // three 16-byte stores into the mapped record
    static_assert(sizeof(TrackIO) == 48 && offsetof(TrackIO, slot) == 32, "TrackIO layout");
    double2* o = reinterpret_cast<double2*>(io_out + t);
    o[0] = make_double2(tx0, ty0);
    o[1] = make_double2(gain, offset);
    reinterpret_cast<int4*>(io_out + t)[2] = make_int4(slot, status, iters, 0);
  }
}

__global__ void k_hypot(const double* x, const double* y, double* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = glibc_hypot(x[i], y[i]);
}

}  // namespace

void debug_hypot(const double* x, const double* y, double* out, int n) {
  if (n <= 0) return;
  const size_t bytes = sizeof(double) * static_cast<size_t>(n);
  double* d = nullptr;
  check_cuda(cudaMalloc(&d, 3 * bytes), "hypot buffers");
  cudaMemcpy(d, x, bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(d + n, y, bytes, cudaMemcpyHostToDevice);
  k_hypot<<<(n + 255) / 256, 256>>>(d, d + n, d + 2 * n, n);
  count_launches(1);
  const cudaError_t e = cudaMemcpy(out, d + 2 * n, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  check_cuda(e, "hypot kernel");
}
}  // namespace lk

namespace {

using Clock = std::chrono::steady_clock;
double us_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::micro>(Clock::now() - t0).count();
}

// cell_candidate_wins (nms.cpp:41-46)
bool wins(const flk_feature& a, const flk_feature& b) {
  if (a.score != b.score) return a.score > b.score;
  if (a.level != b.level) return a.level < b.level;
  if (a.y != b.y) return a.y < b.y;
  return a.x < b.x;
}

int param_dims(ParamMode m) { return m == ParamMode::kTranslation ? 2 : m == ParamMode::kFull ? 4 : 3; }

}  // namespace

Session::Session(const Config& cfg, int device) : cfg_(cfg), device_(device) {
  validate(cfg_);  // frontend.cpp:26-36
  p_ = DetectParams::from(cfg_);
  tp_.mode = static_cast<int>(cfg_.mode);
  tp_.dims = param_dims(cfg_.mode);
  tp_.max_iterations = cfg_.max_iterations;
  tp_.convergence_epsilon = cfg_.convergence_epsilon;
  tp_.min_determinant_factor = 1e-6;  // TrackerConfig default (lk.hpp:44), no config key
}

Session::~Session() {
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  batch_.reset();
  cudaFree(d_frame_);
  cudaFreeHost(h_frame_);
  cudaFree(d_hdr_);
  cudaFree(d_vals_);
  cudaFree(d_coef_);
  cudaFree(d_io_);
  cudaFreeHost(h_io_);
  for (auto ge : graph_exec_)
    if (ge) cudaGraphExecDestroy(ge);
  for (auto e : ev_)
    if (e) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
  if (cur >= 0) cudaSetDevice(cur);
}

void Session::setup(int width, int height) {
  DeviceGuard guard(device_);
  batch_ = std::make_unique<DeviceBatch>(p_, device_, width, height, 1);
  if (!stream_) {
    check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    for (auto& e : ev_) check_cuda(cudaEventCreate(&e), "event");
  }
  pitch_ = (width + 15) & ~15;
  cudaFree(d_frame_);
  cudaFreeHost(h_frame_);
  check_cuda(cudaMalloc(&d_frame_, static_cast<size_t>(pitch_) * height + 16), "frame");
  check_cuda(cudaMallocHost(&h_frame_, static_cast<size_t>(pitch_) * height), "pinned frame");
  // live tracks <= target_count, new candidates <= cells
  const int cells = cols_ * rows_;
  slots_ = cfg_.target_count + cells;
  const size_t L = static_cast<size_t>(batch_->geometry().levels);
  const size_t per = static_cast<size_t>(slots_) * L;
  cudaFree(d_hdr_);
  cudaFree(d_vals_);
  cudaFree(d_coef_);
  cudaFree(d_io_);
  cudaFreeHost(h_io_);
  check_cuda(cudaMalloc(&d_hdr_, per * sizeof(lk::TplLevel)), "templates");
  check_cuda(cudaMalloc(&d_vals_, per * lk::kMaxPx * sizeof(float)), "templates");
  check_cuda(cudaMalloc(&d_coef_, per * lk::kMaxPx * 4 * sizeof(double)), "templates");
  io_bytes_ = kIoHeader + std::max(static_cast<size_t>(slots_) * sizeof(lk::TrackIO),
                                   static_cast<size_t>(slots_) * 3 * sizeof(int) + per * sizeof(int));
  check_cuda(cudaMalloc(&d_io_, io_bytes_), "session io");
  check_cuda(cudaHostAlloc(&h_io_, io_bytes_, cudaHostAllocMapped), "session io (pinned)");
  free_.clear();
  for (int s = slots_ - 1; s >= 0; --s) free_.push_back(s);
  tracks_.clear();
  capture_frame_graph();
}

// The per-frame GPU work as one CUDA graph (replayed with one launch):
// pyramid -> k_track over every slot (CTAs past the live count exit), with
// the stage events inside. The frame and the track records (count in the
// header) are copied ahead of each replay; k_track writes its results into
// the mapped page-locked records. Shapes and pointers are fixed per session.
void Session::capture_frame_graph() {
  for (int timed = 0; timed < 2; ++timed) {
    if (graph_exec_[timed]) cudaGraphExecDestroy(graph_exec_[timed]);
    graph_exec_[timed] = nullptr;
  }
  const Geometry& g = batch_->geometry();
  lk::Levels lv{};
  lv.n = g.levels;
  for (int k = 0; k < g.levels; ++k) {
    lv.img[k] = k == 0 ? d_frame_ : batch_->device_pyramid() + g.loff[k];
    lv.pitch[k] = k == 0 ? pitch_ : g.lpitch[k];
    lv.w[k] = g.lw[k];
    lv.h[k] = g.lh[k];
  }
  const size_t frame_bytes = static_cast<size_t>(pitch_) * g.height;
  uint8_t* m_io = nullptr;
  check_cuda(cudaHostGetDevicePointer(reinterpret_cast<void**>(&m_io), h_io_, 0), "mapped io");
  // two variants: plain, and with stage events (external event-record nodes
  // cost the replay ~20 us, so they are only in the graph used for stats)
  for (int timed = 0; timed < 2; ++timed) {
    auto mark = [&](int i) {
      if (timed)
        check_cuda(cudaEventRecordWithFlags(ev_[i], stream_, cudaEventRecordExternal), "event");
    };
    cudaGraph_t graph = nullptr;
    check_cuda(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
    try {
      // (the frame's H2D and the first stage event are enqueued before each
      // replay: the copy's source is the image itself when it is page-locked)
      graph_launches_ = batch_->enqueue_pyramid(d_frame_, frame_bytes, pitch_, 1, stream_, 0);
      mark(1);
      // k_track writes the results straight into the mapped page-locked
      // mirror: no device-to-host copy to schedule after it
      lk::k_track<<<slots_, 256, 0, stream_>>>(lv, reinterpret_cast<const int*>(d_io_),
                                               reinterpret_cast<const lk::TrackIO*>(d_io_ + kIoHeader),
                                               reinterpret_cast<lk::TrackIO*>(m_io + kIoHeader),
                                               d_hdr_, d_vals_, d_coef_, tp_);
      ++graph_launches_;
      mark(2);
    } catch (...) {
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    check_cuda(cudaStreamEndCapture(stream_, &graph), "end capture");
    const cudaError_t e = cudaGraphInstantiate(&graph_exec_[timed], graph, 0);
    cudaGraphDestroy(graph);
    check_cuda(e, "graph instantiate");
  }
}

void Session::process(const HostImage& img, std::vector<flk_track_info>* out,
                      flk_frame_stats* stats, flk_conformance* conformance) {
  submit(img, stats != nullptr);
  complete(img, out, stats, conformance);
}

// First half of a frame: validation, staging and the frame graph (pyramid +
// LK over the live tracks) enqueued on the session's stream; no host wait.
void Session::submit(const HostImage& img, bool timed) {
  const int cw = cfg_.cell_width(), ch = cfg_.cell_height();
  const int cols = (img.width + cw - 1) / cw, rows = (img.height + ch - 1) / ch;
  if (frame_index_ == 0) {
    width_ = img.width;
    height_ = img.height;
    if (cfg_.target_count > cols * rows)
      throw ConfigError("target count " + std::to_string(cfg_.target_count) + " exceeds the " +
                        std::to_string(cols * rows) + " grid cells of a " +
                        std::to_string(width_) + "x" + std::to_string(height_) + " frame");
  } else if (img.width != width_ || img.height != height_) {
    throw DimensionMismatch("frame " + std::to_string(frame_index_) + " is " +
                            std::to_string(img.width) + "x" + std::to_string(img.height) +
                            ", session expects " + std::to_string(width_) + "x" +
                            std::to_string(height_));
  }
  Geometry::make(p_, img.width, img.height);  // build_pyramid's size rule -> InvalidArgument
  DeviceGuard guard(device_);
  if (!batch_ || batch_->geometry().width != img.width || batch_->geometry().height != img.height) {
    cols_ = cols;
    rows_ = rows;
    setup(img.width, img.height);
  }
  const Geometry& g = batch_->geometry();
  const int L = g.levels;
  flk_frame_stats st{};

  // One submission for the pyramid and the LK launch, one synchronisation:
  // H2D frame, H2D track records, then the graph: pyramid -> k_track (results
  // written to the mapped records).
  // Stage times are CUDA-event device times.
  // one contiguous DMA of the frame at the device pitch, straight from the
  // image's page-locked pixels when the rows already have that pitch, else
  // re-pitched through the pinned staging buffer (a pitched 2-D copy of a
  // small frame costs the copy engine several times longer)
  const uint8_t* src = img.px.data();
  if (!(pitch_ == img.width && img.pinned())) {
    for (int y = 0; y < img.height; ++y)
      std::memcpy(h_frame_ + static_cast<size_t>(y) * pitch_,
                  img.px.data() + static_cast<size_t>(y) * img.width, img.width);
    src = h_frame_;
  }
  if (timed) check_cuda(cudaEventRecord(ev_[0], stream_), "event");
  check_cuda(cudaMemcpyAsync(d_frame_, src, static_cast<size_t>(pitch_) * img.height,
                             cudaMemcpyHostToDevice, stream_), "H2D frame");
  const int n = static_cast<int>(tracks_.size());
  *reinterpret_cast<int*>(h_io_) = n;
  lk::TrackIO* io = reinterpret_cast<lk::TrackIO*>(h_io_ + kIoHeader);
  for (int i = 0; i < n; ++i) {
    std::copy(tracks_[i].warp, tracks_[i].warp + 4, io[i].w);
    io[i].slot = tracks_[i].slot;
  }
  // the live records follow the frame on the copy engine, ahead of the graph
  // (pyramid -> k_track), so the graph holds no copy-engine transitions
  check_cuda(cudaMemcpyAsync(d_io_, h_io_, kIoHeader + sizeof(lk::TrackIO) * static_cast<size_t>(n),
                             cudaMemcpyHostToDevice, stream_), "H2D tracks");
  check_cuda(cudaGraphLaunch(graph_exec_[timed ? 1 : 0], stream_), "frame graph");
  count_launches(graph_launches_);
  submitted_ = true;
}

// Second half: wait for the frame graph, then the lifecycle of
// frontend.cpp:100-225 (retire, trigger, re-detection, dedupe, spawn, output).
void Session::complete(const HostImage& img, std::vector<flk_track_info>* out,
                       flk_frame_stats* stats, flk_conformance* conformance) {
  if (!submitted_) throw InvalidArgument("no submitted frame to complete");
  submitted_ = false;
  DeviceGuard guard(device_);
  const int cw = cfg_.cell_width(), ch = cfg_.cell_height();
  const Geometry& g = batch_->geometry();
  const int L = g.levels;
  flk_frame_stats st{};
  const int n = static_cast<int>(tracks_.size());
  lk::TrackIO* io = reinterpret_cast<lk::TrackIO*>(h_io_ + kIoHeader);
  lk::Levels lv{};
  lv.n = L;
  for (int k = 0; k < L; ++k) {
    lv.img[k] = k == 0 ? d_frame_ : batch_->device_pyramid() + g.loff[k];
    lv.pitch[k] = k == 0 ? pitch_ : g.lpitch[k];
    lv.w[k] = g.lw[k];
    lv.h[k] = g.lh[k];
  }
  check_cuda(cudaStreamSynchronize(stream_), "pyramid + track");
  if (stats) {
    float ms_pyr = 0, ms_trk = 0;
    check_cuda(cudaEventElapsedTime(&ms_pyr, ev_[0], ev_[1]), "stage time");
    check_cuda(cudaEventElapsedTime(&ms_trk, ev_[1], ev_[2]), "stage time");
    st.pyramid_us = ms_pyr * 1e3;
    st.track_us = ms_trk * 1e3;
  }

  // advance live tracks (frontend.cpp:100-131)
  std::vector<flk_track_info> retired;
  st.tracks_entering = n;
  if (n > 0) {
    std::vector<Track> survivors;
    survivors.reserve(tracks_.size());
    for (int i = 0; i < n; ++i) {
      Track& tr = tracks_[i];
      const double* wv = io[i].w;
      st.track_iterations += io[i].iters;
      if (io[i].status == FLK_TRACK_CONVERGED) {
        std::copy(wv, wv + 4, tr.warp);
        survivors.push_back(tr);
      } else {
        retired.push_back(flk_track_info{tr.id, tr.birth.x + wv[0], tr.birth.y + wv[1], wv[2],
                                         wv[3], io[i].status, 0, tr.birth_frame});
        free_.push_back(tr.slot);
      }
    }
    tracks_ = std::move(survivors);
  }
  st.tracks_surviving = static_cast<int>(tracks_.size());

  // trigger rule (frontend.cpp:133-138)
  const int threshold =
      static_cast<int>(std::ceil(cfg_.redetect_ratio * cfg_.target_count - 1e-9));
  st.redetect_fired = st.tracks_surviving < threshold;
  if (conformance) *conformance = flk_conformance{0, 0, 0};

  if (st.redetect_fired) {
    // detection on the pyramid already built
    const auto t0 = Clock::now();
    StageTimes times;
    batch_->run(d_frame_, static_cast<size_t>(pitch_) * img.height, pitch_, 1, stats != nullptr,
                stream_, stats ? &times : nullptr, 0, true);
    std::vector<flk_feature> feats(static_cast<size_t>(g.cells));
    int nf = 0;
    batch_->download(0, 1, &nf, feats.data(), stream_);
    uint64_t dst[2] = {0, 0};
    if (stats)
      check_cuda(cudaMemcpyAsync(dst, batch_->device_stats(), sizeof dst, cudaMemcpyDeviceToHost,
                                 stream_), "D2H stats");
    check_cuda(cudaStreamSynchronize(stream_), "detect");
    feats.resize(static_cast<size_t>(nf));
    const double det_us = us_since(t0);
    st.crf_us = stats ? times.crf_us : det_us;
    st.nms_us = stats ? times.nms_us : 0.0;
    st.nms_candidates = dst[0];
    st.nms_comparisons = dst[1];
    if (conformance)
      *conformance = batch_->conformance(d_frame_, static_cast<size_t>(pitch_) * img.height,
                                         pitch_, stream_);

    // one live track per cell, oldest id wins (frontend.cpp:156-181)
    std::vector<int64_t> occupied;
    std::vector<Track> deduped;
    deduped.reserve(tracks_.size());
    for (Track& tr : tracks_) {
      const double x = tr.birth.x + tr.warp[0], y = tr.birth.y + tr.warp[1];
      const int cx = static_cast<int>(x) / cw, cy = static_cast<int>(y) / ch;
      const int64_t key = static_cast<int64_t>(cy) * g.cols + cx;
      if (std::find(occupied.begin(), occupied.end(), key) == occupied.end()) {
        occupied.push_back(key);
        deduped.push_back(tr);
      } else {
        retired.push_back(flk_track_info{tr.id, x, y, tr.warp[2], tr.warp[3],
                                         FLK_TRACK_CONVERGED, 0, tr.birth_frame});
        free_.push_back(tr.slot);
      }
    }
    tracks_ = std::move(deduped);

    // free cells ranked by cell_candidate_wins (frontend.cpp:183-195)
    std::vector<flk_feature> cands;
    for (const flk_feature& f : feats) {
      const int64_t key = static_cast<int64_t>(f.cell_y) * g.cols + f.cell_x;
      if (std::find(occupied.begin(), occupied.end(), key) == occupied.end()) cands.push_back(f);
    }
    std::sort(cands.begin(), cands.end(), wins);
    const int need = cfg_.target_count - static_cast<int>(tracks_.size());
    if (need > 0 && !cands.empty()) {
      // templates of every ranked candidate in one launch, then the first
      // `need` that build (frontend.cpp:197-210)
      const int nc = static_cast<int>(cands.size());
      int* ci = reinterpret_cast<int*>(h_io_);
      std::vector<int> cslot(nc);
      for (int i = 0; i < nc; ++i) {
        ci[2 * i] = cands[i].x;
        ci[2 * i + 1] = cands[i].y;
        cslot[i] = free_.back();
        free_.pop_back();
        ci[2 * nc + i] = cslot[i];
      }
      int* d_ci = reinterpret_cast<int*>(d_io_);
      check_cuda(cudaMemcpyAsync(d_ci, ci, sizeof(int) * 3 * nc, cudaMemcpyHostToDevice, stream_),
                 "H2D candidates");
      lk::k_template<<<dim3(nc, L), 256, 0, stream_>>>(lv, d_ci, nc, d_hdr_, d_vals_, d_coef_, tp_,
                                                       d_ci + 3 * nc);
      check_cuda(cudaGetLastError(), "k_template");
      count_launches(1);
      int* ts = ci + 3 * nc;
      check_cuda(cudaMemcpyAsync(ts, d_ci + 3 * nc, sizeof(int) * nc * L, cudaMemcpyDeviceToHost,
                                 stream_), "D2H template status");
      check_cuda(cudaStreamSynchronize(stream_), "templates");
      for (int i = 0; i < nc; ++i) {
        bool ok = false, bad = false;
        for (int k = 0; k < L; ++k) {
          const int s = ts[i * L + k];
          ok |= s == 0;
          bad |= s == 1 || s == 2;
        }
        if (static_cast<int>(tracks_.size()) >= cfg_.target_count || bad || !ok) {
          free_.push_back(cslot[i]);
          continue;
        }
        Track tr;
        tr.id = next_id_++;
        tr.birth = cands[i];
        tr.slot = cslot[i];
        tr.warp[0] = tr.warp[1] = tr.warp[2] = tr.warp[3] = 0.0;
        tr.birth_frame = frame_index_;
        tracks_.push_back(tr);
        ++st.tracks_spawned;
      }
    }
    std::sort(tracks_.begin(), tracks_.end(),
              [](const Track& a, const Track& b) { return a.id < b.id; });
  }
  st.feature_count = static_cast<int>(tracks_.size());

  out->clear();
  out->reserve(tracks_.size() + retired.size());
  for (const Track& tr : tracks_)
    out->push_back(flk_track_info{tr.id, tr.birth.x + tr.warp[0], tr.birth.y + tr.warp[1],
                                  tr.warp[2], tr.warp[3], FLK_TRACK_CONVERGED, 1,
                                  tr.birth_frame});
  out->insert(out->end(), retired.begin(), retired.end());
  std::sort(out->begin(), out->end(),
            [](const flk_track_info& a, const flk_track_info& b) { return a.id < b.id; });
  if (stats) *stats = st;
  ++frame_index_;
}

}  // namespace flkb
