"""The C-ABI library loads and exports exactly what include/avion_b200.h declares (no GPU needed)."""

import os
import re

import pytest

from paper_2309_16669_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "avion_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(avb_[a-z0-9_]+)\s*\(", txt))


def test_library_built_and_exports_header():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2309_16669_b200 import build
        build.build()
    lib = _lib.load()
    syms = header_symbols()
    assert syms, "no symbols parsed from header"
    assert syms == set(_lib.EXPORTS), (syms ^ set(_lib.EXPORTS))
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.avb_version() >= 1


def test_host_side_argument_checks_without_gpu():
    lib = _lib.load()
    one = _lib.f32x3([1, 1, 1])
    # bad dims -> AVB_E_ARG before touching any device state
    st = lib.avb_rrc_normalize(None, 1, 0, 10, 10, 0, 0, 0, 0, 0, None, None, None, 4, 4, one, one, 0, 0,
                               None, None)
    assert st == _lib.AVB_E_ARG
    # bad box (host copy given) -> AVB_E_BOX
    import numpy as np
    boxes = np.asarray([[5, 0, 6, 10]], dtype=np.int32)
    st = lib.avb_rrc_normalize(16, 1, 1, 10, 10, 300, 300, 30, 3, 1, 16, None, boxes.ctypes.data, 4, 4, one,
                               one, 0, 0, 16, None)
    assert st == _lib.AVB_E_BOX
    assert b"outside frame" in lib.avb_last_error()
    with pytest.raises(Exception):
        _lib.check(st, "x")
