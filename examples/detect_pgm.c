/*
 * Minimal C caller of the drop-in ABI (the reference README's example,
 * proj/README.md:127-160, unchanged except for the include path):
 *
 *   cc -std=c11 -I include examples/detect_pgm.c -L paper_2003_13493_b200 \
 *      -lfastlk_b200 -Wl,-rpath,$PWD/paper_2003_13493_b200 -o detect_pgm
 *   ./detect_pgm frame.pgm [key=value ...]
 *
 * Prints one "x y score level cell_x cell_y" line per feature, then the
 * frame's counters. Exit code = the failing flk_status.
 */
#include <stdio.h>
#include <string.h>

#include "fastlk.h"

static int fail(flk_status st, const char* what) {
  fprintf(stderr, "%s: %s (%s)\n", what, flk_status_name(st), flk_last_error());
  return (int)st;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s frame.pgm [key=value ...]\n", argv[0]);
    return 1;
  }
  flk_config* cfg = NULL;
  flk_status st = flk_config_create(&cfg);
  if (st != FLK_OK) return fail(st, "config");
  for (int i = 2; i < argc; ++i) {
    char key[64];
    const char* eq = strchr(argv[i], '=');
    if (!eq || (size_t)(eq - argv[i]) >= sizeof key) {
      fprintf(stderr, "bad option %s\n", argv[i]);
      flk_config_destroy(cfg);
      return 1;
    }
    memcpy(key, argv[i], (size_t)(eq - argv[i]));
    key[eq - argv[i]] = '\0';
    if ((st = flk_config_set(cfg, key, eq + 1)) != FLK_OK) {
      flk_config_destroy(cfg);
      return fail(st, argv[i]);
    }
  }
  flk_detector* det = NULL;
  st = flk_detector_create(cfg, &det);
  flk_config_destroy(cfg);
  if (st != FLK_OK) return fail(st, "detector");
  flk_image* img = NULL;
  if ((st = flk_image_load_pgm(argv[1], &img)) != FLK_OK) {
    flk_detector_destroy(det);
    return fail(st, argv[1]);
  }
  flk_features* feats = NULL;
  flk_frame_stats stats;
  st = flk_detector_run(det, img, &feats, &stats, NULL);
  flk_image_destroy(img);
  if (st != FLK_OK) {
    flk_detector_destroy(det);
    return fail(st, "run");
  }
  for (int i = 0; i < flk_features_count(feats); ++i) {
    flk_feature f;
    flk_features_get(feats, i, &f);
    printf("%d %d %.0f %d %d %d\n", f.x, f.y, (double)f.score, f.level, f.cell_x, f.cell_y);
  }
  printf("# features=%d candidates=%llu comparisons=%llu\n", stats.feature_count,
         (unsigned long long)stats.nms_candidates, (unsigned long long)stats.nms_comparisons);
  flk_features_destroy(feats);
  flk_detector_destroy(det);
  return 0;
}
