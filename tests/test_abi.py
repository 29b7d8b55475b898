"""The drop-in boundary on CPU (no GPU needed): the library loads, exports
every symbol the headers declare, and its host-side behaviour (status codes,
config parsing, validation order, PGM I/O, NULL handling) matches the
reference C ABI called with the same arguments (proj/tests/test_capi.cpp).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2003_13493_b200 as fl
from paper_2003_13493_b200 import fastlk as fk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    names = []
    for h in ("fastlk.h", "fastlk_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"FLK_API\s+[\w\s\*]+?\b(flkb?_\w+)\s*\(", text)
    return names


def test_library_exports_every_declared_symbol():
    lib = fk.load_library()
    names = header_symbols()
    assert len(names) == len(set(names)) and len(names) >= 44
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(fk.ABI_SYMBOLS + fk.EXT_SYMBOLS)


def test_reference_abi_is_a_subset():
    """Every flk_* symbol the reference header declares is exported here."""
    ref_h = "/root/reference/proj/include/fastlk/fastlk.h"
    if not os.path.exists(ref_h):
        pytest.skip("reference header not mounted on this box")
    ref = set(re.findall(r"FLK_API\s+[\w\s\*]+?\b(flk_\w+)\s*\(", open(ref_h).read()))
    assert len(ref) == 26
    assert ref <= set(header_symbols())


def test_status_names_and_version():
    assert fl.status_name(0) == "ok"
    assert fl.status_name(2) == "io error"
    assert fl.version() == "0.1.0"
    lib = fk.load_library()
    assert lib.flk_track_status_name(0) == b"CONVERGED"
    assert lib.flk_track_status_name(3) == b"SINGULAR_HESSIAN"


def test_null_arguments_rejected_with_message():
    lib = fk.load_library()
    assert lib.flk_image_load_pgm(None, None) == fk.FLK_E_INVALID_ARG
    assert len(lib.flk_last_error()) > 0
    assert lib.flk_config_create(None) == fk.FLK_E_INVALID_ARG
    assert lib.flk_detector_create(None, None) == fk.FLK_E_INVALID_ARG
    assert lib.flk_detector_run(None, None, None, None, None) == fk.FLK_E_INVALID_ARG
    assert lib.flk_features_count(None) == 0 and lib.flk_image_width(None) == 0
    lib.flk_features_destroy(None)
    lib.flk_image_destroy(None)


def _ref_lib():
    import oracle
    if oracle.load_reference() is None:
        pytest.skip("reference build unavailable")
    lib = ctypes.CDLL(oracle.REF_LIB)
    lib.flk_config_create.argtypes = [ctypes.POINTER(ctypes.c_void_p)]
    lib.flk_config_set.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_char_p]
    lib.flk_config_load_file.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
    lib.flk_detector_create.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    lib.flk_detector_destroy.argtypes = [ctypes.c_void_p]
    lib.flk_config_destroy.argtypes = [ctypes.c_void_p]
    lib.flk_image_load_pgm.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    lib.flk_image_destroy.argtypes = [ctypes.c_void_p]
    lib.flk_image_width.argtypes = [ctypes.c_void_p]
    return lib


CONFIG_CASES = [
    ("epsilon", "12"), ("epsilon", " 12"), ("epsilon", "12 "), ("epsilon", "twelve"),
    ("epsilon", "+7"), ("epsilon", "-3"), ("epsilon", "1e3"), ("epsilon", "99999999999"),
    ("N", "9"), ("N", "20"), ("score_kind", "mt"), ("score_kind", "MT"), ("score_kind", "sad_a"),
    ("l", "3"), ("w", "0"), ("h", "8"), ("n", "0"), ("threads", "8"), ("target_count", "0"),
    ("redetect_ratio", "0.5"), ("redetect_ratio", "1.0"), ("redetect_ratio", "abc"),
    ("param_mode", "translation_gain"), ("param_mode", "affine"), ("max_iterations", "0"),
    ("convergence_epsilon", "0"), ("convergence_epsilon", "1e-3"), ("bogus", "1"), ("", "1"),
]


@pytest.mark.parametrize("key,value", CONFIG_CASES)
def test_config_set_and_validation_match_reference(key, value):
    """flk_config_set status, then flk_detector_create's validation status,
    are the reference's for the same single-key change (config.cpp:70-131,
    frontend.cpp:26-36). On a box without a GPU our create stops at
    FLK_E_INTERNAL only after validation passed."""
    ref = _ref_lib()
    lib = fk.load_library()
    results = []
    for L in (ref, lib):
        c = ctypes.c_void_p()
        assert L.flk_config_create(ctypes.byref(c)) == 0
        s1 = L.flk_config_set(c, key.encode(), value.encode())
        d = ctypes.c_void_p()
        s2 = L.flk_detector_create(c, ctypes.byref(d))
        if s2 == 0:
            L.flk_detector_destroy(d)
        L.flk_config_destroy(c)
        results.append((s1, s2))
    (r1, r2), (o1, o2) = results
    assert o1 == r1
    if r2 != 0:
        assert o2 == r2
    else:
        assert o2 in (0, fk.FLK_E_INTERNAL)


def test_config_file_matches_reference(tmp_path):
    ref = _ref_lib()
    lib = fk.load_library()
    files = {
        "ok.cfg": "# comment\n\nepsilon = 12\nN=9\n  score_kind =  mt  \nl = 3\nh = 8\n",
        "bad_line.cfg": "epsilon 12\n",
        "empty_value.cfg": "epsilon =\n",
        "unknown.cfg": "eps = 3\n",
        "bad_int.cfg": "n = x\n",
    }
    for name, text in files.items():
        p = tmp_path / name
        p.write_text(text)
        st = []
        for L in (ref, lib):
            c = ctypes.c_void_p()
            L.flk_config_create(ctypes.byref(c))
            st.append(L.flk_config_load_file(c, str(p).encode()))
            L.flk_config_destroy(c)
        assert st[0] == st[1], name
    c = fl.Config()
    with pytest.raises(fl.IoError):
        c.load_file(str(tmp_path / "missing.cfg"))


def test_pgm_io_matches_reference(tmp_path):
    ref = _ref_lib()
    lib = fk.load_library()
    cases = {
        "ok.pgm": b"P5\n4 2\n255\n" + bytes(range(8)),
        "comment.pgm": b"P5\n# generated\n2 # w then h\n1\n255\n\x07\x09",
        "ascii.pgm": b"P2\n2 2\n255\n0 0 0 0\n",
        "maxval.pgm": b"P5\n2 2\n65535\n\x00",
        "trunc.pgm": b"P5\n4 4\n255\nab",
        "zero.pgm": b"P5\n0 4\n255\n",
        "badint.pgm": b"P5\n4x 4\n255\n",
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        out = []
        for L in (ref, lib):
            h = ctypes.c_void_p()
            s = L.flk_image_load_pgm(str(p).encode(), ctypes.byref(h))
            w = L.flk_image_width(h) if s == 0 else -1
            if s == 0:
                L.flk_image_destroy(h)
            out.append((s, w))
        assert out[0] == out[1], name
    img = fl.Image.load_pgm(str(tmp_path / "comment.pgm"))
    assert (img.width, img.height) == (2, 1)
    arr = np.arange(37 * 21, dtype=np.uint8).reshape(21, 37)
    fl.Image.from_array(arr).save_pgm(str(tmp_path / "rt.pgm"))
    raw = (tmp_path / "rt.pgm").read_bytes()
    assert raw.startswith(b"P5\n37 21\n255\n") and raw.endswith(arr.tobytes())


def test_image_errors():
    with pytest.raises(fl.InvalidArgument):
        fl.Image.from_array(np.zeros((0, 4), np.uint8))
    with pytest.raises(fl.IoError) as e:
        fl.Image.load_pgm("missing_file.pgm")
    assert "missing_file.pgm" in str(e.value)


def test_session_create_validates_before_the_device():
    """flk_session_create: NULL checks, then the reference's config validation
    (frontend.cpp:26-36: ratio / target -> FLK_E_CONFIG, tracker ranges ->
    FLK_E_INVALID_ARG), then the device (no CPU fallback)."""
    import torch
    lib = fk.load_library()
    s = ctypes.c_void_p()
    assert lib.flk_session_create(None, ctypes.byref(s)) == fk.FLK_E_INVALID_ARG
    for key, val, code in (("redetect_ratio", "1.0", fk.FLK_E_CONFIG),
                           ("target_count", "0", fk.FLK_E_CONFIG),
                           ("max_iterations", "0", fk.FLK_E_INVALID_ARG),
                           ("convergence_epsilon", "0", fk.FLK_E_INVALID_ARG)):
        c = fl.Config().set(key, val)
        assert lib.flk_session_create(c.handle, ctypes.byref(s)) == code
    if not torch.cuda.is_available():
        assert lib.flk_session_create(fl.Config().handle, ctypes.byref(s)) == fk.FLK_E_INTERNAL
        assert b"no CPU fallback" in lib.flk_last_error()


def test_no_cpu_fallback_without_gpu():
    """On a box without a CUDA device the detector refuses loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(fl.InternalError) as e:
        fl.Detector(fl.Config())
    assert "no CPU fallback" in str(e.value)
