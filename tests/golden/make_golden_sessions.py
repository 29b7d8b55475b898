"""Regenerate tests/golden/sessions.json from the UNMODIFIED reference.

Run in the build container (needs /root/reference or oracle/_ref):
    python tests/golden/make_golden_sessions.py
Every tests/cases.py SESSIONS entry is run through the reference's own
flk_session_* C ABI (oracle/_ref/libfastlk_ref.so); per frame the SHA-256 of
the track records (id, x, y, alpha, beta, status, live, birth_frame), their
count and the deterministic flk_frame_stats counters are stored.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import sessions  # noqa: E402
from cases import SESSIONS  # noqa: E402


def main():
    ref = oracle.load_reference()
    assert ref is not None, "reference build unavailable"
    out = {}
    for name, kind, n, w, h, cfg in SESSIONS:
        frames = sessions.sequence(kind, n, w, h)
        res = sessions.run_capi_session(ref.lib, cfg, frames)
        out[name] = dict(sequence=kind, frames_n=n, width=w, height=h, config=cfg,
                         frames=sessions.digest(res))
        print(name, [r[1]["feature_count"] for r in res])
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sessions.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
