/*
 * TEST INFRASTRUCTURE ONLY -- CPU parity oracle for the tracking session
 * (SURVEY §8(f) rows f1 re-detection masking/ranking and f2 pyramidal LK).
 *
 * A plain-C restatement of the reference's inverse-compositional LK tracker
 * (src/fastlk/lk.cpp) and of the detect-track lifecycle Frontend::
 * process_frame (src/fastlk/frontend.cpp:65-225) that the CUDA session is
 * checked against. Double arithmetic is written in the reference's order:
 * compiled without contraction (-std=c11 implies -ffp-contract=off; no -mfma),
 * every sum is the reference's serial sum, so the results are bit-identical
 * to the reference build (pinned in tests/test_oracle_lk.py). Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load it.
 *
 * Paths are relative to /root/reference/proj.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fastlk_oracle.h"

/* ------------------------------------------------------------ primitives */

/* sample_bilinear (src/fastlk/image.cpp:67-81); the caller guarantees the
 * position is inside the image (the reference throws otherwise). */
static float sample_bilinear(const uint8_t* img, int w, int h, double x, double y) {
  const int x0 = (int)x;
  const int y0 = (int)y;
  const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
  const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
  const double fx = x - x0;
  const double fy = y - y0;
  const double top = (1.0 - fx) * img[(size_t)y0 * w + x0] + fx * img[(size_t)y0 * w + x1];
  const double bot = (1.0 - fx) * img[(size_t)y1 * w + x0] + fx * img[(size_t)y1 * w + x1];
  return (float)((1.0 - fy) * top + fy * bot);
}

int orc_param_dims(int mode) {
  /* param_dims (lk.cpp:50-58) */
  switch (mode) {
    case ORC_MODE_TRANSLATION: return 2;
    case ORC_MODE_TRANSLATION_OFFSET: return 3;
    case ORC_MODE_TRANSLATION_GAIN: return 3;
    default: return 4;
  }
}
static int has_gain(int mode) { return mode == ORC_MODE_TRANSLATION_GAIN || mode == ORC_MODE_FULL; }
static int has_offset(int mode) {
  return mode == ORC_MODE_TRANSLATION_OFFSET || mode == ORC_MODE_FULL;
}

/* det_small (lk.cpp:74-102): LU with partial pivoting, n-stride layout. */
static double det_small(const double* in, int n) {
  double m[16];
  memcpy(m, in, sizeof m);
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

/* invert_small (lk.cpp:105-143): Gauss-Jordan with partial pivoting. */
static int invert_small(const double* in, int n, double* out) {
  double m[16], inv[16];
  memcpy(m, in, sizeof m);
  memset(inv, 0, sizeof inv);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int row = col + 1; row < n; ++row)
      if (fabs(m[row * n + col]) > fabs(m[pivot * n + col])) pivot = row;
    const double p = m[pivot * n + col];
    if (p == 0.0) return 0;
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
  memcpy(out, inv, sizeof inv);
  return 1;
}

void orc_default_tracker(orc_tracker* t) {
  /* TrackerConfig defaults (lk.hpp:40-48) */
  t->mode = ORC_MODE_FULL;
  t->max_iterations = 30;
  t->convergence_epsilon = 0.01;
  t->min_determinant_factor = 1e-6;
}

int orc_validate_tracker(const orc_tracker* t) {
  /* validate(TrackerConfig) (lk.cpp:37-47) */
  if (t->max_iterations < 1) return ORC_E_INVALID_ARG;
  if (!(t->convergence_epsilon > 0.0)) return ORC_E_INVALID_ARG;
  if (!(t->min_determinant_factor > 0.0)) return ORC_E_INVALID_ARG;
  return ORC_OK;
}

static int patch_size(int level) { return level <= 1 ? 16 : 8; }

/* ------------------------------------------------------ build_template */

/* build_template (lk.cpp:147-240). */
int orc_build_template(const uint8_t* const* lv, const int* wk, const int* hk, int nlevels,
                       int fx0, int fy0, const orc_tracker* cfg, orc_templates* out) {
  memset(out, 0, sizeof *out);
  for (int k = 0; k < nlevels; ++k) {
    const int w = wk[k], h = hk[k];
    const int patch = patch_size(k);
    if (w < patch + 2 || h < patch + 2) continue;
    const int half = patch / 2;
    const double ax = fx0 / (double)(1 << k);
    const double ay = fy0 / (double)(1 << k);
    if (ax - half - 1 < 0.0 || ax + half > w - 1 || ay - half - 1 < 0.0 || ay + half > h - 1) {
      out->error = ORC_TPL_OUT_OF_BOUNDS;
      out->nlevels = 0;
      return ORC_OK;
    }
    orc_patch* t = &out->lv[out->nlevels];
    t->level = k;
    t->patch = patch;
    t->anchor_x = ax;
    t->anchor_y = ay;
    t->dims = orc_param_dims(cfg->mode);
    const int dims = t->dims;
    double hess[16] = {0};
    int idx = 0;
    for (int oy = -half; oy < half; ++oy) {
      for (int ox = -half; ox < half; ++ox, ++idx) {
        const double px = ax + ox;
        const double py = ay + oy;
        const float value = sample_bilinear(lv[k], w, h, px, py);
        const float gx = 0.5f * (sample_bilinear(lv[k], w, h, px + 1, py) -
                                 sample_bilinear(lv[k], w, h, px - 1, py));
        const float gy = 0.5f * (sample_bilinear(lv[k], w, h, px, py + 1) -
                                 sample_bilinear(lv[k], w, h, px, py - 1));
        t->values[idx] = value;
        double* u = &t->coeffs[idx * dims];
        u[0] = gx;
        u[1] = gy;
        int d = 2;
        if (has_gain(cfg->mode)) u[d++] = value;
        if (has_offset(cfg->mode)) u[d++] = 1.0;
        for (int r = 0; r < dims; ++r)
          for (int c = 0; c < dims; ++c) hess[r * dims + c] += u[r] * u[c];
      }
    }
    t->hessian_det = det_small(hess, dims);
    const double area = (double)(patch * patch);
    if (!(t->hessian_det >= cfg->min_determinant_factor * area * area) ||
        !invert_small(hess, dims, t->hessian_inv)) {
      out->error = ORC_TPL_SINGULAR;
      out->nlevels = 0;
      return ORC_OK;
    }
    out->nlevels++;
  }
  if (out->nlevels == 0) out->error = ORC_TPL_OUT_OF_BOUNDS;
  return ORC_OK;
}

/* ------------------------------------------------------- track_feature */

/* track_feature (lk.cpp:242-350); the residual is not observable through the
 * C ABI and is not computed. */
int orc_track_feature(const orc_templates* tpls, const uint8_t* const* lv, const int* wk,
                      const int* hk, int nlevels, const double* init, const orc_tracker* cfg,
                      orc_track_result* res) {
  if (tpls->error != ORC_TPL_OK || tpls->nlevels == 0) return ORC_E_INVALID_ARG;
  double tx0 = init[0], ty0 = init[1], gain = init[2], offset = init[3];
  int aborted = 0, finest_converged = 0;
  res->status = ORC_TRACK_CONVERGED;
  res->iterations = 0;
  for (int li = tpls->nlevels - 1; li >= 0; --li) {
    const orc_patch* t = &tpls->lv[li];
    if (t->level >= nlevels) return ORC_E_INVALID_ARG;
    const uint8_t* img = lv[t->level];
    const int w = wk[t->level], h = hk[t->level];
    const double scale = (double)(1 << t->level);
    double tx = tx0 / scale;
    double ty = ty0 / scale;
    const int half = t->patch / 2;
    const int dims = t->dims;
    const double max_step = 0.5 * hypot(w, h);
    int level_converged = 0;
    for (int iter = 0; iter < cfg->max_iterations; ++iter) {
      const double bx0 = t->anchor_x - half + tx;
      const double bx1 = t->anchor_x + half - 1 + tx;
      const double by0 = t->anchor_y - half + ty;
      const double by1 = t->anchor_y + half - 1 + ty;
      if (bx0 < 0.0 || by0 < 0.0 || bx1 > w - 1 || by1 > h - 1) {
        res->status = ORC_TRACK_OUT_OF_BOUNDS;
        aborted = 1;
        break;
      }
      double rhs[4] = {0, 0, 0, 0};
      int idx = 0;
      for (int oy = -half; oy < half; ++oy) {
        for (int ox = -half; ox < half; ++ox, ++idx) {
          const double sample =
              sample_bilinear(img, w, h, t->anchor_x + ox + tx, t->anchor_y + oy + ty);
          const double r = sample - (1.0 + gain) * t->values[idx] - offset;
          const double* u = &t->coeffs[idx * dims];
          for (int d = 0; d < dims; ++d) rhs[d] += u[d] * r;
        }
      }
      double delta[4] = {0, 0, 0, 0};
      for (int r = 0; r < dims; ++r) {
        double acc = 0.0;
        for (int c = 0; c < dims; ++c) acc += t->hessian_inv[r * dims + c] * rhs[c];
        delta[r] = acc;
      }
      res->iterations++;
      tx -= delta[0];
      ty -= delta[1];
      int d = 2;
      if (has_gain(cfg->mode)) gain += delta[d++];
      if (has_offset(cfg->mode)) offset += delta[d++];
      const double step = hypot(delta[0], delta[1]);
      if (step > max_step || !(gain > -1.0) || !isfinite(step)) {
        res->status = ORC_TRACK_DIVERGED;
        aborted = 1;
        break;
      }
      if (step <= cfg->convergence_epsilon) {
        level_converged = 1;
        break;
      }
    }
    tx0 = tx * scale;
    ty0 = ty * scale;
    if (aborted) break;
    if (li == 0) finest_converged = level_converged;
  }
  res->warp[0] = tx0;
  res->warp[1] = ty0;
  res->warp[2] = gain;
  res->warp[3] = offset;
  if (!aborted && !finest_converged) res->status = ORC_TRACK_MAX_ITERATIONS;
  return ORC_OK;
}

/* ------------------------------------------------------------- session */

typedef struct track {
  int64_t id;
  orc_feature birth;
  orc_templates* tpl;
  double warp[4];
  int birth_frame;
} track;

struct orc_session {
  orc_session_cfg cfg;
  track* tracks;  /* ascending id */
  int ntracks, cap;
  int64_t next_id;
  int frame_index, width, height;
};

int orc_session_create(const orc_session_cfg* cfg, orc_session** out) {
  /* Frontend::Frontend -> validate(FrontendConfig) (frontend.cpp:26-36) */
  int st = orc_validate(&cfg->det);
  if (st == ORC_OK) st = orc_validate_tracker(&cfg->tracker);
  if (st != ORC_OK) return st;
  if (cfg->target_count < 1) return ORC_E_CONFIG;
  if (!(cfg->redetect_ratio > 0.0 && cfg->redetect_ratio < 1.0)) return ORC_E_CONFIG;
  orc_session* s = (orc_session*)calloc(1, sizeof *s);
  s->cfg = *cfg;
  *out = s;
  return ORC_OK;
}

void orc_session_destroy(orc_session* s) {
  if (!s) return;
  for (int i = 0; i < s->ntracks; ++i) free(s->tracks[i].tpl);
  free(s->tracks);
  free(s);
}

/* cell_candidate_wins (nms.cpp:41-46) as a qsort comparator: winners first. */
static int cand_cmp(const void* pa, const void* pb) {
  const orc_feature* a = (const orc_feature*)pa;
  const orc_feature* b = (const orc_feature*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  if (a->level != b->level) return a->level < b->level ? -1 : 1;
  if (a->y != b->y) return a->y < b->y ? -1 : 1;
  if (a->x != b->x) return a->x < b->x ? -1 : 1;
  return 0;
}

static int obs_cmp(const void* pa, const void* pb) {
  const orc_track_info* a = (const orc_track_info*)pa;
  const orc_track_info* b = (const orc_track_info*)pb;
  return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

static void push_track(orc_session* s, const track* t) {
  if (s->ntracks == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 64;
    s->tracks = (track*)realloc(s->tracks, (size_t)s->cap * sizeof(track));
  }
  s->tracks[s->ntracks++] = *t;
}

/* Frontend::process_frame (frontend.cpp:65-225). out must hold every live
 * and retired track of the frame (at most live tracks + target_count). */
int orc_session_process(orc_session* s, const uint8_t* img, int width, int height,
                        orc_track_info* out, int cap, int* count, orc_session_stats* stats,
                        orc_conformance* conf) {
  const orc_params* p = &s->cfg.det;
  const int cw = orc_cell_width(p), ch = orc_cell_height(p);
  const int cols = (width + cw - 1) / cw, rows = (height + ch - 1) / ch;
  memset(stats, 0, sizeof *stats);
  if (conf) memset(conf, 0, sizeof *conf);
  if (s->frame_index == 0) {
    s->width = width;
    s->height = height;
    if (s->cfg.target_count > cols * rows) return ORC_E_CONFIG;
  } else if (width != s->width || height != s->height) {
    return ORC_E_DIMENSION;
  }
  const int L = p->num_levels;
  int wk[16], hk[16];
  if (orc_pyramid_dims(width, height, L, wk, hk) != ORC_OK) return ORC_E_INVALID_ARG;
  size_t total = 0;
  for (int k = 0; k < L; ++k) total += (size_t)wk[k] * hk[k];
  uint8_t* pyr = (uint8_t*)malloc(total);
  orc_build_pyramid(img, width, height, L, pyr);
  const uint8_t* lv[16];
  size_t off = 0;
  for (int k = 0; k < L; ++k) {
    lv[k] = pyr + off;
    off += (size_t)wk[k] * hk[k];
  }

  int nret = 0, nout = 0;
  orc_track_info* retired = (orc_track_info*)malloc(sizeof(orc_track_info) * (size_t)(s->ntracks + 1));
  /* advance live tracks (frontend.cpp:100-131) */
  stats->tracks_entering = s->ntracks;
  {
    int keep = 0;
    for (int i = 0; i < s->ntracks; ++i) {
      track* t = &s->tracks[i];
      orc_track_result r;
      orc_track_feature(t->tpl, lv, wk, hk, L, t->warp, &s->cfg.tracker, &r);
      stats->track_iterations += r.iterations;
      if (r.status == ORC_TRACK_CONVERGED) {
        memcpy(t->warp, r.warp, sizeof t->warp);
        s->tracks[keep++] = *t;
      } else {
        orc_track_info o = {t->id, t->birth.x + r.warp[0], t->birth.y + r.warp[1], r.warp[2],
                            r.warp[3], r.status, 0, t->birth_frame};
        retired[nret++] = o;
        free(t->tpl);
      }
    }
    s->ntracks = keep;
  }
  stats->tracks_surviving = s->ntracks;
  const int threshold = (int)ceil(s->cfg.redetect_ratio * s->cfg.target_count - 1e-9);
  stats->redetect_fired = s->ntracks < threshold;

  if (stats->redetect_fired) {
    orc_feature* feats = (orc_feature*)malloc(sizeof(orc_feature) * (size_t)(cols * rows));
    int nf = 0;
    orc_stats ds;
    orc_detect(img, width, height, p, feats, cols * rows, &nf, &ds);
    stats->nms_comparisons = ds.comparisons;
    stats->nms_candidates = ds.candidates;
    if (conf) orc_conformance_check(img, width, height, p, feats, nf, conf);
    /* one live track per cell, oldest id wins (frontend.cpp:162-181); the
     * reference keys an unordered_set by cy*cols+cx, emulated as a list */
    long* keys = (long*)malloc(sizeof(long) * (size_t)(s->ntracks + 1));
    int nkeys = 0;
    retired = (orc_track_info*)realloc(retired, sizeof(orc_track_info) * (size_t)(nret + s->ntracks + 1));
    int keep = 0;
    for (int i = 0; i < s->ntracks; ++i) {
      track* t = &s->tracks[i];
      const double x = t->birth.x + t->warp[0], y = t->birth.y + t->warp[1];
      const int cx = (int)x / cw, cy = (int)y / ch;
      const long key = (long)cy * cols + cx;
      int seen = 0;
      for (int j = 0; j < nkeys && !seen; ++j) seen = keys[j] == key;
      if (!seen) {
        keys[nkeys++] = key;
        s->tracks[keep++] = *t;
      } else {
        orc_track_info o = {t->id, x, y, t->warp[2], t->warp[3], ORC_TRACK_CONVERGED, 0,
                            t->birth_frame};
        retired[nret++] = o;
        free(t->tpl);
      }
    }
    s->ntracks = keep;
    /* free cells ranked by cell_candidate_wins (frontend.cpp:183-195) */
    int nc = 0;
    for (int i = 0; i < nf; ++i) {
      const long key = (long)feats[i].cell_y * cols + feats[i].cell_x;
      int seen = 0;
      for (int j = 0; j < nkeys && !seen; ++j) seen = keys[j] == key;
      if (!seen) feats[nc++] = feats[i];
    }
    qsort(feats, (size_t)nc, sizeof(orc_feature), cand_cmp);
    for (int i = 0; i < nc; ++i) {
      if (s->ntracks >= s->cfg.target_count) break;
      orc_templates* tpl = (orc_templates*)malloc(sizeof(orc_templates));
      orc_build_template(lv, wk, hk, L, feats[i].x, feats[i].y, &s->cfg.tracker, tpl);
      if (tpl->error != ORC_TPL_OK || tpl->nlevels == 0) {
        free(tpl);
        continue;
      }
      track t;
      t.id = s->next_id++;
      t.birth = feats[i];
      t.tpl = tpl;
      t.warp[0] = t.warp[1] = t.warp[2] = t.warp[3] = 0.0;
      t.birth_frame = s->frame_index;
      push_track(s, &t);
      stats->tracks_spawned++;
    }
    free(keys);
    free(feats);
  }
  stats->feature_count = s->ntracks;
  for (int i = 0; i < s->ntracks && nout < cap; ++i) {
    const track* t = &s->tracks[i];
    orc_track_info o = {t->id, t->birth.x + t->warp[0], t->birth.y + t->warp[1], t->warp[2],
                        t->warp[3], ORC_TRACK_CONVERGED, 1, t->birth_frame};
    out[nout++] = o;
  }
  for (int i = 0; i < nret && nout < cap; ++i) out[nout++] = retired[i];
  qsort(out, (size_t)nout, sizeof(orc_track_info), obs_cmp);
  *count = nout;
  free(retired);
  free(pyr);
  s->frame_index++;
  return ORC_OK;
}
