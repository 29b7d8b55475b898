// Detection conformance on the device -- the reference's flk_detector_run
// fills `flk_conformance` by re-running a deliberately naive detector
// (oracle.cpp:37-161 per-pixel labels, rotation-scan arc test, linear-scan
// MT, run-scan SAD-A; oracle.cpp:173-200 raster suppression) and tallying
// the emitted features against it (oracle.cpp:240-268). These kernels are
// that naive detector, written independently of the fast path's bit
// algebra so the tally stays a real cross-check. They run only when the
// caller passes a non-NULL conformance pointer.
#pragma once

#include <cstdint>

#include "fast_math.cuh"

namespace flkb {

__device__ __forceinline__ bool naive_arc(const int (&lab)[16], int which, int n) {
  for (int s = 0; s < 16; ++s) {
    bool ok = true;
    for (int j = 0; j < n && ok; ++j) ok = lab[(s + j) & 15] == which;
    if (ok) return true;
  }
  return false;
}

__device__ float naive_pixel(const uint8_t* p, int pitch, int eps, int n, int kind) {
  int c = p[0], ring[16], lab[16];
  for (int i = 0; i < 16; ++i) {
    ring[i] = p[ring_dy(i) * pitch + ring_dx(i)];
    lab[i] = ring[i] < c - eps ? -1 : (ring[i] > c + eps ? 1 : 0);
  }
  if (!naive_arc(lab, -1, n) && !naive_arc(lab, 1, n)) return 0.0f;
  if (kind == kSadB) {
    long sum = 0;
    for (int i = 0; i < 16; ++i) {
      const int d = abs(ring[i] - c);
      if (d > eps) sum += d - eps;
    }
    return static_cast<float>(sum);
  }
  if (kind == kSadA) {
    long best = -1;
    for (int pol = -1; pol <= 1; pol += 2) {
      if (!naive_arc(lab, pol, n)) continue;
      bool all = true;
      for (int i = 0; i < 16; ++i) all = all && lab[i] == pol;
      for (int s = 0; s < 16; ++s) {
        if (!all && !(lab[s] == pol && lab[(s + 15) & 15] != pol)) continue;
        if (all && s > 0) break;
        int len = 0;
        long sum = 0;
        while (len < 16 && lab[(s + len) & 15] == pol) {
          sum += max(abs(ring[(s + len) & 15] - c) - eps, 0);
          ++len;
        }
        if (len >= n && sum > best) best = sum;
      }
    }
    return best < 0 ? 0.0f : static_cast<float>(best);
  }
  int mt = eps;
  for (int e = eps; e <= 255; ++e) {
    int l2[16];
    for (int i = 0; i < 16; ++i) l2[i] = ring[i] < c - e ? -1 : (ring[i] > c + e ? 1 : 0);
    if (naive_arc(l2, -1, n) || naive_arc(l2, 1, n)) mt = e;
    else break;
  }
  return static_cast<float>(mt);
}

__global__ void k_naive_fast(const uint8_t* img, int pitch, int w, int h, int eps, int n,
                             int kind, float* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  float s = 0.0f;
  if (x >= 3 && x < w - 3 && y >= 3 && y < h - 3)
    s = naive_pixel(img + static_cast<size_t>(y) * pitch + x, pitch, eps, n, kind);
  out[static_cast<size_t>(y) * w + x] = s;
}

__device__ __forceinline__ bool naive_survives(const float* r, int w, int h, int x, int y, int n) {
  const float s = r[static_cast<size_t>(y) * w + x];
  if (s <= 0.0f) return false;
  for (int dy = -n; dy <= n; ++dy)
    for (int dx = -n; dx <= n; ++dx) {
      if (!dx && !dy) continue;
      const int nx = x + dx, ny = y + dy;
      if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
      const float v = r[static_cast<size_t>(ny) * w + nx];
      if (v > s || (v == s && (ny < y || (ny == y && nx < x)))) return false;
    }
  return true;
}

__global__ void k_naive_survivors(const float* r, int w, int h, int n, int* total) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  if (naive_survives(r, w, h, x, y, n)) atomicAdd(total, 1);
}

// conf[0] = naive survivors, conf[1] = matched, conf[2] = false positives
__global__ void k_conf_features(const flk_feature* feats, const int* count,
                                const float* const* maps, const int* lw, const int* lh, int n,
                                int* conf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *count) return;
  const flk_feature ft = feats[i];
  const int k = ft.level, lx = ft.x >> k, ly = ft.y >> k;
  const float* r = maps[k];
  if (r[static_cast<size_t>(ly) * lw[k] + lx] <= 0.0f) {
    atomicAdd(conf + 2, 1);
    return;
  }
  if (naive_survives(r, lw[k], lh[k], lx, ly, n)) atomicAdd(conf + 1, 1);
}

}  // namespace flkb
