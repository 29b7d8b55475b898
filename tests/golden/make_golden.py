"""Regenerate tests/golden/golden.npz + golden.json from the UNMODIFIED reference.

Run in the build container (needs /root/reference or oracle/_ref):
    python tests/golden/make_golden.py
Each case in tests/cases.py is detected by oracle/_ref/libfastlk_ref.so
(the reference's own detect_frame + C-ABI flatten, or the reference's own
primitives composed at the extension cell size); the feature list and the
deterministic counters are stored. Large cases store a SHA-256 of the feature
bytes instead of the list.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import synth  # noqa: E402
from cases import GOLDEN  # noqa: E402


def main():
    ref = oracle.load_reference()
    assert ref is not None, "reference build unavailable"
    arrays, meta = {}, {}
    for name, fam, f, w, h, cfg, full in GOLDEN:
        img = synth.frame(fam, f, w, h)
        p = oracle.make_params(**cfg)
        feats, st = ref.detect(img, p)
        meta[name] = dict(family=fam, frame=f, width=w, height=h, config=cfg,
                          count=int(len(feats)), comparisons=int(st.comparisons),
                          candidates=int(st.candidates),
                          sha256=hashlib.sha256(feats.tobytes()).hexdigest(),
                          image_sha256=hashlib.sha256(img.tobytes()).hexdigest(),
                          full=bool(full))
        if full:
            arrays[name] = feats
        print(name, len(feats), st.candidates, st.comparisons)
    here = os.path.dirname(os.path.abspath(__file__))
    np.savez_compressed(os.path.join(here, "golden.npz"), **arrays)
    with open(os.path.join(here, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
