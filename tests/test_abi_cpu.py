"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports every symbol
include/jit_sched.h declares (no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "jit_sched.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jit_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("jit_sched_init", "jit_sched_step", "jit_sched_replay", "jit_sched_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2504_20068_b200 import _build
    path = _build.build_library()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    lib.jit_sched_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.jit_sched_version()


def test_binding_names_match_header():
    from paper_2504_20068_b200 import jitsched
    assert sorted(jitsched.EXPORTS) == _declared()


def test_product_path_does_not_touch_oracle():
    """The product package never imports or links the oracle (it must fail loudly, not fall back)."""
    pkg = os.path.join(ROOT, "paper_2504_20068_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".inc", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "from oracle" not in txt, f


def test_workspace_query_rejects_bad_config():
    from paper_2504_20068_b200 import jitsched
    import numpy as np
    import workloads as W
    lib = jitsched.load_library()
    cfg = jitsched.make_config(W.default_config(prefill_chunk=10 ** 6), 128, 4)
    edges = np.arange(1, 9, dtype=np.uint32)
    cum = np.zeros((1, 8), np.uint32)
    t = jitsched.jit_len_table(1, 8, 8, 0, edges.ctypes.data, cum.ctypes.data)
    n = ctypes.c_uint64()
    assert lib.jit_sched_workspace_bytes(ctypes.byref(cfg), ctypes.byref(t), ctypes.byref(n)) == -1
    cfg = jitsched.make_config(W.default_config(), 128, 4)
    assert lib.jit_sched_workspace_bytes(ctypes.byref(cfg), ctypes.byref(t), ctypes.byref(n)) == 0
    assert n.value > 128 * 32
