/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference detector
 * hot path, used as the parity checker for the CUDA product. See
 * fastlk_oracle.h for how it is pinned to the reference. Citations are
 * file:line into /root/reference/proj.
 */
#include "fastlk_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ parameters */

void orc_default_params(orc_params* p) {
  /* Defaults of FastParams / GridConfig (fast.hpp:20-24, nms.hpp:17-22). */
  p->epsilon = 10;
  p->arc_length = 10;
  p->score_kind = ORC_SAD_B;
  p->num_levels = 1;
  p->cell_width_units = 1;
  p->cell_height_units = 32;
  p->nms_radius = 1;
  p->cell_width_px = 0;
  p->cell_height_px = 0;
}

/* validate(FastParams) fast.cpp:18-27 and validate(GridConfig) nms.cpp:13-23. */
int orc_validate(const orc_params* p) {
  if (p->epsilon < 0 || p->epsilon > 255) return ORC_E_INVALID_ARG;
  if (p->arc_length < 9 || p->arc_length > 16) return ORC_E_INVALID_ARG;
  if (p->score_kind < ORC_SAD_B || p->score_kind > ORC_MT) return ORC_E_INVALID_ARG;
  if (p->cell_width_units < 1 || p->cell_height_units < 1) return ORC_E_INVALID_ARG;
  if (p->num_levels < 1) return ORC_E_INVALID_ARG;
  if (p->nms_radius < 1) return ORC_E_INVALID_ARG;
  if (p->cell_width_px < 0 || p->cell_height_px < 0) return ORC_E_INVALID_ARG;
  return ORC_OK;
}

/* GridConfig::cell_width / cell_height (nms.hpp:23-24). */
int orc_cell_width(const orc_params* p) {
  return p->cell_width_px > 0 ? p->cell_width_px : 32 * p->cell_width_units;
}
int orc_cell_height(const orc_params* p) {
  return p->cell_height_px > 0 ? p->cell_height_px
                               : (1 << (p->num_levels - 1)) * p->cell_height_units;
}

/* ---------------------------------------------------------------- pyramid */

/* Size checks of build_pyramid (image.cpp:37-45); dims floor-halve (:52). */
int orc_pyramid_dims(int width, int height, int levels, int* wk, int* hk) {
  if (levels < 1 || width < 1 || height < 1) return ORC_E_INVALID_ARG;
  int mn = width < height ? width : height;
  if ((mn >> (levels - 1)) < 8) return ORC_E_INVALID_ARG;
  int w = width, h = height;
  for (int k = 0; k < levels; ++k) {
    wk[k] = w;
    hk[k] = h;
    w /= 2;
    h /= 2;
  }
  return ORC_OK;
}

/* Cascaded 2x2 round-half-up mean, each level from the previous rounded one
 * (image.cpp:49-62). */
int orc_build_pyramid(const uint8_t* img, int width, int height, int levels,
                      uint8_t* out) {
  int wk[32], hk[32];
  if (levels > 32) return ORC_E_INVALID_ARG;
  int rc = orc_pyramid_dims(width, height, levels, wk, hk);
  if (rc) return rc;
  memcpy(out, img, (size_t)width * height);
  const uint8_t* src = out;
  uint8_t* dst = out + (size_t)width * height;
  for (int k = 1; k < levels; ++k) {
    const int sw = wk[k - 1];
    for (int y = 0; y < hk[k]; ++y) {
      const uint8_t* r0 = src + (size_t)(2 * y) * sw;
      const uint8_t* r1 = r0 + sw;
      for (int x = 0; x < wk[k]; ++x) {
        int s = r0[2 * x] + r0[2 * x + 1] + r1[2 * x] + r1[2 * x + 1];
        dst[(size_t)y * wk[k] + x] = (uint8_t)((s + 2) >> 2);
      }
    }
    src = dst;
    dst += (size_t)wk[k] * hk[k];
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------- FAST */

/* kBresenhamCircle (fast.cpp:13-16): clockwise from (0,-3), y down. */
static const int kRing[16][2] = {
    {0, -3}, {1, -3}, {2, -2}, {3, -1}, {3, 0}, {3, 1}, {2, 2}, {1, 3},
    {0, 3}, {-1, 3}, {-2, 2}, {-3, 1}, {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3}};

/* has_cyclic_run (fast.cpp:37-48): doubled-word scan for the longest run. */
int orc_has_cyclic_run(uint16_t mask, int min_len) {
  if (mask == 0xFFFFu) return min_len <= 16;
  uint32_t d = ((uint32_t)mask << 16) | mask;
  int run = 0, best = 0;
  for (int i = 0; i < 32; ++i) {
    if ((d >> i) & 1u) {
      ++run;
      if (run > best) best = run;
    } else {
      run = 0;
    }
  }
  return best >= min_len;
}

/* arc_oracle (oracle.cpp:15-25): try all 16 rotations. */
int orc_arc_oracle(uint16_t mask, int min_len) {
  if (min_len <= 0) return 1;
  if (min_len > 16) return 0;
  uint32_t want = (min_len == 16) ? 0xFFFFu : ((1u << min_len) - 1u);
  uint32_t m = mask;
  for (int r = 0; r < 16; ++r) {
    uint32_t rot = ((m >> r) | (m << (16 - r))) & 0xFFFFu;
    if ((rot & want) == want) return 1;
  }
  return 0;
}

/* 8 KB bit table per arc length (fast.cpp:52-65), built lazily. */
static uint32_t g_lut[17][2048];
static int g_lut_ready[17];

static const uint32_t* lut_for(int n) {
  if (!g_lut_ready[n]) {
    memset(g_lut[n], 0, sizeof(g_lut[n]));
    for (uint32_t m = 0; m <= 0xFFFFu; ++m)
      if (orc_has_cyclic_run((uint16_t)m, n)) g_lut[n][m >> 5] |= 1u << (m & 31u);
    g_lut_ready[n] = 1;
  }
  return g_lut[n];
}

static int lut_test(const uint32_t* lut, uint16_t m) {
  return (lut[m >> 5] >> (m & 31u)) & 1u;
}

typedef struct sample {
  int c;
  int ring[16];
} sample;

/* masks_at (fast.cpp:98-111). */
static void masks(const sample* s, int eps, uint16_t* dark, uint16_t* bright) {
  int lo = s->c - eps, hi = s->c + eps;
  uint16_t d = 0, b = 0;
  for (int i = 0; i < 16; ++i) {
    if (s->ring[i] < lo) d |= (uint16_t)(1u << i);
    if (s->ring[i] > hi) b |= (uint16_t)(1u << i);
  }
  *dark = d;
  *bright = b;
}

static int term(const sample* s, int i, int eps) {
  int d = abs(s->ring[i] - s->c) - eps;
  return d > 0 ? d : 0;
}

/* best_arc_sum (fast.cpp:123-154): best sum over maximal runs >= min_len. */
static long best_arc(uint16_t mask, int min_len, const sample* s, int eps) {
  if (mask == 0) return -1;
  if (mask == 0xFFFFu) {
    long sum = 0;
    for (int i = 0; i < 16; ++i) sum += term(s, i, eps);
    return min_len > 16 ? -1 : sum;
  }
  int start = 0;
  while ((mask >> start) & 1u) ++start;
  long best = -1, run_sum = 0;
  int run_len = 0;
  for (int step = 1; step <= 16; ++step) {
    int i = (start + step) & 15;
    if ((mask >> i) & 1u) {
      ++run_len;
      run_sum += term(s, i, eps);
      if (run_len >= min_len && run_sum > best) best = run_sum;
    } else {
      run_len = 0;
      run_sum = 0;
    }
  }
  return best;
}

/* max_threshold_score (fast.cpp:168-181): binary search on [eps, 255]. */
static int max_threshold(const sample* s, int eps, const uint32_t* lut) {
  int lo = eps, hi = 255;
  while (lo < hi) {
    int mid = (lo + hi + 1) / 2;
    uint16_t d, b;
    masks(s, mid, &d, &b);
    if (lut_test(lut, d) || lut_test(lut, b))
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

/* score_sample (fast.cpp:183-203). */
static float score_sample(const sample* s, uint16_t dark, uint16_t bright,
                          const orc_params* p, const uint32_t* lut) {
  switch (p->score_kind) {
    case ORC_SAD_B: {
      long sum = 0;
      for (int i = 0; i < 16; ++i) sum += term(s, i, p->epsilon);
      return (float)sum;
    }
    case ORC_SAD_A: {
      long best = -1, v;
      if (lut_test(lut, dark)) {
        v = best_arc(dark, p->arc_length, s, p->epsilon);
        if (v > best) best = v;
      }
      if (lut_test(lut, bright)) {
        v = best_arc(bright, p->arc_length, s, p->epsilon);
        if (v > best) best = v;
      }
      return best < 0 ? 0.0f : (float)best;
    }
    default:
      return (float)max_threshold(s, p->epsilon, lut);
  }
}

/* score_at (fast.cpp:221-247): cardinal pretest, masks, two LUT probes. */
static float score_at(const uint8_t* img, int w, int x, int y,
                      const orc_params* p, const uint32_t* lut) {
  const uint8_t* px = img + (size_t)y * w + x;
  int c = px[0];
  int lo = c - p->epsilon, hi = c + p->epsilon;
  int v0 = px[kRing[0][1] * w + kRing[0][0]];
  int v4 = px[kRing[4][1] * w + kRing[4][0]];
  int v8 = px[kRing[8][1] * w + kRing[8][0]];
  int v12 = px[kRing[12][1] * w + kRing[12][0]];
  int nd = (v0 < lo) + (v4 < lo) + (v8 < lo) + (v12 < lo);
  int nb = (v0 > hi) + (v4 > hi) + (v8 > hi) + (v12 > hi);
  if (nd < 2 && nb < 2) return 0.0f;
  sample s;
  s.c = c;
  for (int i = 0; i < 16; ++i) s.ring[i] = px[kRing[i][1] * w + kRing[i][0]];
  uint16_t d, b;
  masks(&s, p->epsilon, &d, &b);
  if (!lut_test(lut, d) && !lut_test(lut, b)) return 0.0f;
  return score_sample(&s, d, b, p, lut);
}

/* detect_responses for one level (fast.cpp:273-303): 3-px border stays 0. */
int orc_fast_level(const uint8_t* img, int w, int h, const orc_params* p,
                   float* resp) {
  int rc = orc_validate(p);
  if (rc) return rc;
  const uint32_t* lut = lut_for(p->arc_length);
  memset(resp, 0, sizeof(float) * (size_t)w * h);
  if (h - 6 <= 0 || w <= 6) return ORC_OK;
  for (int y = 3; y < h - 3; ++y)
    for (int x = 3; x < w - 3; ++x)
      resp[(size_t)y * w + x] = score_at(img, w, x, y, p, lut);
  return ORC_OK;
}

/* corner_score (fast.cpp:267-271) for an interior pixel. */
float orc_corner_score(const uint8_t* img, int w, int h, int x, int y,
                       const orc_params* p) {
  if (x < 3 || x >= w - 3 || y < 3 || y >= h - 3) return -1.0f;
  const uint32_t* lut = lut_for(p->arc_length);
  sample s;
  s.c = img[(size_t)y * w + x];
  for (int i = 0; i < 16; ++i)
    s.ring[i] = img[(size_t)(y + kRing[i][1]) * w + x + kRing[i][0]];
  uint16_t d, b;
  masks(&s, p->epsilon, &d, &b);
  if (!lut_test(lut, d) && !lut_test(lut, b)) return 0.0f;
  return score_sample(&s, d, b, p, lut);
}

/* -------------------------------------------------------------------- NMS */

/* cell_candidate_wins (nms.cpp:41-46). */
static int wins(const orc_feature* a, const orc_feature* b) {
  if (a->score != b->score) return a->score > b->score;
  if (a->level != b->level) return a->level < b->level;
  if (a->y != b->y) return a->y < b->y;
  return a->x < b->x;
}

/* spiral_is_local_max (nms.cpp:48-79): ring walk top, right, bottom, left;
 * counts in-image neighbours up to and including the first suppressor. */
static int spiral(const float* r, int w, int h, int x, int y, int radius,
                  uint64_t* comparisons) {
  const float s = r[(size_t)y * w + x];
  uint64_t count = 0;
  int lost = 0;
#define ORC_VISIT(nx, ny)                                                   \
  do {                                                                      \
    int nx_ = (nx), ny_ = (ny);                                             \
    if (nx_ >= 0 && ny_ >= 0 && nx_ < w && ny_ < h) {                       \
      ++count;                                                              \
      float v = r[(size_t)ny_ * w + nx_];                                   \
      if (v > s || (v == s && (ny_ < y || (ny_ == y && nx_ < x)))) lost = 1; \
    }                                                                       \
  } while (0)
  for (int rr = 1; rr <= radius && !lost; ++rr) {
    for (int dx = -rr; dx <= rr && !lost; ++dx) ORC_VISIT(x + dx, y - rr);
    for (int dy = -rr + 1; dy <= rr && !lost; ++dy) ORC_VISIT(x + rr, y + dy);
    for (int dx = rr - 1; dx >= -rr && !lost; --dx) ORC_VISIT(x + dx, y + rr);
    for (int dy = rr - 1; dy >= -rr + 1 && !lost; --dy) ORC_VISIT(x - rr, y + dy);
  }
#undef ORC_VISIT
  if (comparisons) *comparisons += count;
  return !lost;
}

/* suppress_and_select (nms.cpp:81-135): every positive pixel of every level
 * that survives its own level's spiral test competes for its projected cell. */
int orc_suppress_and_select(const float* const* resp, const int* wk,
                            const int* hk, const orc_params* p,
                            orc_feature* cells, int* cols, int* rows,
                            orc_stats* stats) {
  int rc = orc_validate(p);
  if (rc) return rc;
  const int cw = orc_cell_width(p), ch = orc_cell_height(p);
  *cols = (wk[0] + cw - 1) / cw;
  *rows = (hk[0] + ch - 1) / ch;
  const int n = (*cols) * (*rows);
  for (int i = 0; i < n; ++i) cells[i].level = -1;
  for (int k = 0; k < p->num_levels; ++k) {
    const float* r = resp[k];
    for (int y = 0; y < hk[k]; ++y) {
      for (int x = 0; x < wk[k]; ++x) {
        float s = r[(size_t)y * wk[k] + x];
        if (s <= 0.0f) continue;
        if (stats) ++stats->candidates;
        if (!spiral(r, wk[k], hk[k], x, y, p->nms_radius,
                    stats ? &stats->comparisons : NULL))
          continue;
        orc_feature c;
        c.x = x << k; /* rescale_to_level0, nms.hpp:67-69 */
        c.y = y << k;
        c.score = s;
        c.level = k;
        c.cell_x = c.x / cw;
        c.cell_y = c.y / ch;
        orc_feature* slot = &cells[(size_t)c.cell_y * (*cols) + c.cell_x];
        if (slot->level < 0 || wins(&c, slot)) *slot = c;
      }
    }
  }
  return ORC_OK;
}

/* detect_frame (frontend.cpp:38-57) + flatten (capi.cpp:260-269). */
int orc_detect(const uint8_t* img, int width, int height, const orc_params* p,
               orc_feature* out, int cap, int* count, orc_stats* stats) {
  int rc = orc_validate(p);
  if (rc) return rc;
  int wk[32], hk[32];
  if (p->num_levels > 32) return ORC_E_INVALID_ARG;
  rc = orc_pyramid_dims(width, height, p->num_levels, wk, hk);
  if (rc) return rc;
  size_t total = 0;
  for (int k = 0; k < p->num_levels; ++k) total += (size_t)wk[k] * hk[k];
  uint8_t* pyr = (uint8_t*)malloc(total);
  float* resp_all = (float*)malloc(sizeof(float) * total);
  const float* resp[32];
  orc_build_pyramid(img, width, height, p->num_levels, pyr);
  size_t off = 0;
  for (int k = 0; k < p->num_levels; ++k) {
    orc_fast_level(pyr + off, wk[k], hk[k], p, resp_all + off);
    resp[k] = resp_all + off;
    off += (size_t)wk[k] * hk[k];
  }
  const int cw = orc_cell_width(p), ch = orc_cell_height(p);
  const int ncell = ((width + cw - 1) / cw) * ((height + ch - 1) / ch);
  orc_feature* cells = (orc_feature*)malloc(sizeof(orc_feature) * (size_t)ncell);
  int cols, rows;
  if (stats) memset(stats, 0, sizeof(*stats));
  orc_suppress_and_select(resp, wk, hk, p, cells, &cols, &rows, stats);
  int nf = 0;
  for (int i = 0; i < cols * rows; ++i) {
    if (cells[i].level < 0) continue;
    if (nf < cap) out[nf] = cells[i];
    ++nf;
  }
  *count = nf;
  if (stats) stats->feature_count = nf;
  free(cells);
  free(resp_all);
  free(pyr);
  return nf > cap ? ORC_E_INVALID_ARG : ORC_OK;
}

/* ------------------------------------------------------------ conformance */

/* naive_score (oracle.cpp:109-148): explicit labels, rotation scan, MT by a
 * linear scan. Independent of the LUT path above. */
static int naive_has_arc(const int* lab, int which, int n) {
  for (int s = 0; s < 16; ++s) {
    int ok = 1;
    for (int j = 0; j < n && ok; ++j) ok = lab[(s + j) & 15] == which;
    if (ok) return 1;
  }
  return 0;
}

static void naive_label(const uint8_t* img, int w, int x, int y, int eps,
                        int* c, int* ring, int* lab) {
  *c = img[(size_t)y * w + x];
  for (int i = 0; i < 16; ++i) {
    int v = img[(size_t)(y + kRing[i][1]) * w + x + kRing[i][0]];
    ring[i] = v;
    lab[i] = v < *c - eps ? -1 : (v > *c + eps ? 1 : 0);
  }
}

static float naive_score(const uint8_t* img, int w, int x, int y,
                         const orc_params* p) {
  int c, ring[16], lab[16];
  naive_label(img, w, x, y, p->epsilon, &c, ring, lab);
  int dark = naive_has_arc(lab, -1, p->arc_length);
  int bright = naive_has_arc(lab, 1, p->arc_length);
  if (!dark && !bright) return 0.0f;
  if (p->score_kind == ORC_SAD_B) {
    long sum = 0;
    for (int i = 0; i < 16; ++i) {
      int d = abs(ring[i] - c);
      if (d > p->epsilon) sum += d - p->epsilon;
    }
    return (float)sum;
  }
  if (p->score_kind == ORC_SAD_A) {
    long best = -1;
    for (int pol = -1; pol <= 1; pol += 2) {
      if (!naive_has_arc(lab, pol, p->arc_length)) continue;
      int all = 1;
      for (int i = 0; i < 16; ++i) all &= lab[i] == pol;
      if (all) {
        long sum = 0;
        for (int i = 0; i < 16; ++i) {
          int d = abs(ring[i] - c) - p->epsilon;
          sum += d > 0 ? d : 0;
        }
        if (sum > best) best = sum;
        continue;
      }
      for (int s = 0; s < 16; ++s) {
        if (!(lab[s] == pol && lab[(s + 15) & 15] != pol)) continue;
        int len = 0;
        long sum = 0;
        while (len < 16 && lab[(s + len) & 15] == pol) {
          int d = abs(ring[(s + len) & 15] - c) - p->epsilon;
          sum += d > 0 ? d : 0;
          ++len;
        }
        if (len >= p->arc_length && sum > best) best = sum;
      }
    }
    return best < 0 ? 0.0f : (float)best;
  }
  int mt = p->epsilon;
  for (int e = p->epsilon; e <= 255; ++e) {
    int c2, r2[16], l2[16];
    naive_label(img, w, x, y, e, &c2, r2, l2);
    if (naive_has_arc(l2, -1, p->arc_length) || naive_has_arc(l2, 1, p->arc_length))
      mt = e;
    else
      break;
  }
  return (float)mt;
}

/* raster_local_max_mask (oracle.cpp:173-200). */
static int raster_survives(const float* r, int w, int h, int x, int y, int n) {
  float s = r[(size_t)y * w + x];
  if (s <= 0.0f) return 0;
  for (int dy = -n; dy <= n; ++dy)
    for (int dx = -n; dx <= n; ++dx) {
      if (!dx && !dy) continue;
      int nx = x + dx, ny = y + dy;
      if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
      float v = r[(size_t)ny * w + nx];
      if (v > s || (v == s && (ny < y || (ny == y && nx < x)))) return 0;
    }
  return 1;
}

/* conformance_check (oracle.cpp:240-268). */
int orc_conformance_check(const uint8_t* img, int width, int height,
                    const orc_params* p, const orc_feature* feats, int count,
                    orc_conformance* out) {
  int wk[32], hk[32];
  if (p->num_levels > 32) return ORC_E_INVALID_ARG;
  int rc = orc_pyramid_dims(width, height, p->num_levels, wk, hk);
  if (rc) return rc;
  size_t total = 0;
  for (int k = 0; k < p->num_levels; ++k) total += (size_t)wk[k] * hk[k];
  uint8_t* pyr = (uint8_t*)malloc(total);
  float* resp = (float*)calloc(total, sizeof(float));
  orc_build_pyramid(img, width, height, p->num_levels, pyr);
  size_t offs[32];
  size_t off = 0;
  long survivors = 0;
  for (int k = 0; k < p->num_levels; ++k) {
    offs[k] = off;
    for (int y = 3; y < hk[k] - 3; ++y)
      for (int x = 3; x < wk[k] - 3; ++x)
        resp[off + (size_t)y * wk[k] + x] = naive_score(pyr + off, wk[k], x, y, p);
    for (int y = 0; y < hk[k]; ++y)
      for (int x = 0; x < wk[k]; ++x)
        survivors += raster_survives(resp + off, wk[k], hk[k], x, y, p->nms_radius);
    off += (size_t)wk[k] * hk[k];
  }
  out->matched = out->false_positives = 0;
  for (int i = 0; i < count; ++i) {
    int k = feats[i].level;
    int lx = feats[i].x >> k, ly = feats[i].y >> k;
    const float* r = resp + offs[k];
    if (r[(size_t)ly * wk[k] + lx] <= 0.0f) {
      ++out->false_positives;
      continue;
    }
    if (raster_survives(r, wk[k], hk[k], lx, ly, p->nms_radius)) ++out->matched;
  }
  out->subset_only = (int)survivors - out->matched;
  free(resp);
  free(pyr);
  return ORC_OK;
}

/* -------------------------------------------------------- synthetic frames */

/* counter hash h(f,i,salt) = splitmix64(SEED ^ f<<32 ^ i ^ salt<<60). */
static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t synth_hash(uint64_t f, uint64_t i, uint64_t salt) {
  return splitmix64(0x200313493ull ^ (f << 32) ^ i ^ (salt << 60));
}

void orc_synth_frame(int kind, uint64_t frame, int width, int height,
                     uint8_t* out) {
  if (kind == 0) {
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x)
        out[(size_t)y * width + x] =
            (uint8_t)(synth_hash(frame, (uint64_t)y * width + x, 0) & 0xFF);
    return;
  }
  const uint64_t gw = (uint64_t)(width / 8 + 2);
  for (int y = 0; y < height; ++y) {
    for (int x = 0; x < width; ++x) {
      uint64_t gx = (uint64_t)(x >> 3), gy = (uint64_t)(y >> 3);
      int64_t v00 = 30 + (int64_t)(synth_hash(frame, gy * gw + gx, 1) % 160);
      int64_t v10 = 30 + (int64_t)(synth_hash(frame, gy * gw + gx + 1, 1) % 160);
      int64_t v01 = 30 + (int64_t)(synth_hash(frame, (gy + 1) * gw + gx, 1) % 160);
      int64_t v11 = 30 + (int64_t)(synth_hash(frame, (gy + 1) * gw + gx + 1, 1) % 160);
      int64_t wx = (x & 7) * 32, wy = (y & 7) * 32;
      int64_t top = v00 * (256 - wx) + v10 * wx;
      int64_t bot = v01 * (256 - wx) + v11 * wx;
      int64_t val = (top * (256 - wy) + bot * wy + 32768) >> 16;
      val += (int64_t)(synth_hash(frame, (uint64_t)y * width + x, 2) % 7) - 3;
      if (val < 0) val = 0;
      if (val > 255) val = 255;
      out[(size_t)y * width + x] = (uint8_t)val;
    }
  }
}
