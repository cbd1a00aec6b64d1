"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h
declares, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1805_06124_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rbg():
    B.build()
    from paper_1805_06124_b200 import rbg as R
    return R


def declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(rbg_\w+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(rbg):
    names = declared_functions()
    assert {"rbg_create", "rbg_run", "rbg_destroy", "rbg_get_basis", "rbg_gen_chirp"} <= names
    L = ctypes.CDLL(rbg.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n
    assert set(rbg.SYMBOLS) == names


def test_lanes_match_design(rbg):
    # DESIGN.md fixes L_S = 32, L_I = 2048; the oracle's CANONICAL constant is written
    # independently from the same document.
    from oracle import oracle as O
    assert rbg.lanes() == O.CANONICAL
    assert "L_S=32" in rbg.version()


def _create(rbg, S, w, tol, k_max, dtype):
    h = ctypes.c_void_p()
    st = rbg.lib().rbg_create(ctypes.byref(h), S.ctypes.data if S is not None else None,
                              S.shape[1] if S is not None else 4, S.shape[0] if S is not None else 4,
                              w.ctypes.data if w is not None else None, tol, k_max, dtype)
    return st, rbg.lib().rbg_last_error().decode()


@pytest.mark.parametrize("case", ["kmax0", "kmax_big", "tol_neg", "tol_nan", "w_zero", "w_nan",
                                  "null_S", "dtype"])
def test_invalid_arguments_rejected(rbg, case):
    S = np.ones((5, 4))                   # M = 5 columns of N = 4
    w = np.ones(4)
    tol, k_max, dtype = 0.0, 3, rbg.REAL_F64
    if case == "kmax0":
        k_max = 0
    elif case == "kmax_big":
        k_max = 5                          # > N = 4
    elif case == "tol_neg":
        tol = -1.0
    elif case == "tol_nan":
        tol = float("nan")
    elif case == "w_zero":
        w = np.array([1.0, 0.0, 1.0, 1.0])
    elif case == "w_nan":
        w = np.array([1.0, np.nan, 1.0, 1.0])
    elif case == "null_S":
        S = None
    elif case == "dtype":
        dtype = 7
    st, msg = _create(rbg, S, w, tol, k_max, dtype)
    assert st == rbg.EINVAL, (st, msg)


def test_destroy_null_is_safe(rbg):
    rbg.lib().rbg_destroy(None)


def test_python_binding_has_every_c_name(rbg):
    """The thin binding offers every entry point under the C name without its `rbg_` prefix."""
    missing = [n for n in declared_functions() if not callable(getattr(rbg, n[len("rbg_"):], None))]
    assert not missing, missing
