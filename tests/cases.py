"""Parity cases: (image family, frame, size, detector config).

Named after BASELINE.json's configs: C1..C5 plus edge
cases (S3). Config keys are the reference's (config.cpp:70-131); cw/ch are the
B200 extension's cell-size override in pixels (0 = reference geometry).
Test infrastructure only.
"""

def _cfg(epsilon=10, N=9, score_kind="sad_b", l=1, w=1, h=32, n=1, cw=0, ch=0):
    return dict(epsilon=epsilon, N=N, score_kind=score_kind, l=l, w=w, h=h, n=n,
                cell_width_px=cw, cell_height_px=ch)


# (name, family, frame index, width, height, config, store_full)
GOLDEN = []
for fam in ("noise", "texture"):
    for kind in ("mt", "sad_b"):
        GOLDEN.append((f"C1_{fam}_{kind}", fam, 0, 752, 480, _cfg(score_kind=kind), True))
    for f in (0, 1):
        for kind in ("sad_b", "sad_a", "mt"):
            GOLDEN.append((f"C2_{fam}_f{f}_{kind}", fam, f, 752, 480,
                           _cfg(score_kind=kind, l=3, h=8), True))
GOLDEN += [
    ("C3_texture_16x16", "texture", 0, 1920, 1080, _cfg(N=12, l=4, cw=16, ch=16), False),
    ("C3_texture_32x16", "texture", 0, 1920, 1080, _cfg(N=12, l=4, h=2), False),
    ("C3_noise_16x16", "noise", 0, 1920, 1080, _cfg(N=12, l=4, cw=16, ch=16), False),
    ("C5_texture_4k", "texture", 0, 3840, 2160, _cfg(N=10, l=5, h=2), False),
    ("odd_753x481_l3", "texture", 2, 753, 481, _cfg(l=3, h=8), True),
    ("odd_753x481_noise_n2", "noise", 2, 753, 481, _cfg(l=3, h=8, n=2, score_kind="sad_a"), True),
    ("smallest_32x32_l3", "noise", 4, 32, 32, _cfg(l=3, h=8), True),
    ("smallest_8x8", "noise", 5, 8, 8, _cfg(), True),
    ("eps0_mt", "texture", 3, 200, 150, _cfg(epsilon=0, score_kind="mt", l=2, h=16), True),
    ("eps255", "noise", 3, 200, 150, _cfg(epsilon=255, l=2, h=16), True),
    ("eps250_N16_noise", "noise", 6, 200, 150, _cfg(epsilon=40, N=16, l=2, h=16), True),
    ("quant4_n1", "quant4", 0, 256, 192, _cfg(l=2, h=16), True),
    ("quant4_n3_mt", "quant4", 1, 256, 192, _cfg(l=2, h=16, n=3, score_kind="mt"), True),
    ("quant4_n4_sada", "quant4", 2, 256, 192, _cfg(l=3, h=8, n=4, score_kind="sad_a"), True),
    ("blocks_ties", "blocks", 0, 320, 240, _cfg(l=3, h=8, n=2), True),
    ("constant", "constant", 0, 128, 96, _cfg(l=2, h=16), True),
    ("capi_like_256x192", "texture", 10, 256, 192, _cfg(N=10, l=2, h=16), True),
    ("wide_cells_w2", "texture", 7, 500, 300, _cfg(N=11, l=2, w=2, h=8), True),
    ("tall_cells_h3_l4", "noise", 8, 400, 300, _cfg(N=10, l=4, w=3, h=3), True),
    ("N12_mt_l2", "texture", 9, 640, 360, _cfg(N=12, l=2, h=16, score_kind="mt"), True),
    ("N16_sada", "texture", 11, 300, 200, _cfg(epsilon=5, N=16, l=1, score_kind="sad_a"), True),
    ("ext_8x8_cells", "texture", 12, 256, 128, _cfg(l=2, cw=8, ch=8), True),
]


# Tracking sessions (SURVEY §8(f) f1 + f2): (name, sequence, frames, width,
# height, flk_config entries). Sequences come from tests/sessions.py.
def _scfg(l=2, h=16, target=100, ratio=0.3, mode="full", iters=30, conv=0.01, **det):
    c = dict(epsilon=10, N=9, score_kind="sad_b", l=l, w=1, h=h, n=1, target_count=target,
             redetect_ratio=ratio, param_mode=mode, max_iterations=iters,
             convergence_epsilon=conv)
    c.update(det)
    return c


SESSIONS = [
    ("slide_512x256_l2", "slide3", 48, 512, 256, _scfg()),
    ("drift_320x240_l3_full", "drift", 16, 320, 240, _scfg(l=3, h=8, target=60, ratio=0.5)),
    ("drift_translation", "drift", 10, 256, 192, _scfg(target=40, mode="translation")),
    ("drift_offset", "drift", 10, 256, 192, _scfg(target=40, mode="translation_offset")),
    ("drift_gain_mt", "drift", 10, 256, 192, _scfg(target=40, mode="translation_gain",
                                                 score_kind="mt", N=10)),
    ("slide_maxit2", "slide5", 12, 320, 192, _scfg(target=50, iters=2, conv=0.001,
                                                   ratio=0.9)),
    ("noise_l3_n2", "noise", 6, 256, 192, _scfg(l=3, h=8, target=40, n=2)),
    ("c2_752x480_l3", "slide2", 8, 752, 480, _scfg(l=3, h=8, target=200, ratio=0.6)),
    ("c2_752x480_l3_long", "slide2", 40, 752, 480, _scfg(l=3, h=8, target=200, ratio=0.3)),
    ("drift_l4_w2_h4_sada", "drift", 12, 640, 480, _scfg(l=4, w=2, h=4, target=50, ratio=0.7,
                                                         score_kind="sad_a", N=11)),
]
