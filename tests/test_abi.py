"""The C-ABI library loads without a GPU and exports every symbol include/sketchycgal.h declares."""
import os
import re

import paper_1912_02949_b200 as scg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sketchycgal.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sketchycgal_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    scg.build()
    lib = scg.open_library(scg.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(scg.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", scg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_rejects_bad_arguments_without_gpu():
    import ctypes
    import numpy as np
    lib = scg.open_library(scg.LIB_PATH)
    rp = np.array([0, 1, 2], dtype=np.int64)
    col = np.array([0, 1], dtype=np.int32)
    val = np.array([1.0, 1.0])
    csr = scg.Csr(2, 0, 2, rp.ctypes.data, col.ctypes.data, val.ctypes.data, 1)
    h = ctypes.c_void_p()
    # R > n, alpha <= 0, beta0 <= 0 are argument errors (SCG_EINVAL) checked before touching the device
    assert lib.sketchycgal_maxcut_init(ctypes.byref(h), ctypes.byref(csr), 3, 2.0, 1.0, 0, 1, None, 0, None) == -1
    assert lib.sketchycgal_maxcut_init(ctypes.byref(h), ctypes.byref(csr), 1, 0.0, 1.0, 0, 1, None, 0, None) == -1
    assert lib.sketchycgal_maxcut_init(ctypes.byref(h), ctypes.byref(csr), 1, 2.0, -1.0, 0, 1, None, 0, None) == -1
    bad = np.array([1, 0], dtype=np.int32)  # columns not ascending
    rp2 = np.array([0, 2, 2], dtype=np.int64)
    csr2 = scg.Csr(2, 0, 2, rp2.ctypes.data, bad.ctypes.data, val.ctypes.data, 1)
    assert lib.sketchycgal_maxcut_init(ctypes.byref(h), ctypes.byref(csr2), 1, 2.0, 1.0, 0, 1, None, 0, None) == -1
    assert not h.value
