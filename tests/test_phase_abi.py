"""The phase retrieval C-ABI library (include/scg_phase.h) builds for sm_100a, loads without a GPU,
exports every declared symbol and rejects bad arguments before touching the device."""
import ctypes
import os
import re
import subprocess

import numpy as np

from paper_1912_02949_b200 import phase as pr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "scg_phase.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scg_pr_\w+)\s*\(", src)))


def test_phase_library_exports_every_declared_symbol():
    pr.build()
    lib = pr.open_library(pr.PHASE_LIB)
    declared = _declared()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(pr.EXPORTS) == declared


def test_phase_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", pr.PHASE_LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_phase_init_rejects_bad_arguments_without_gpu():
    lib = pr.open_library(pr.PHASE_LIB)
    h = ctypes.c_void_p()

    def init(n, L, R, alpha=3.0, beta0=1.0, psi=None):
        psi = np.ones((L, n), dtype=np.complex128) if psi is None else psi
        b = np.ones((L, n))
        return lib.scg_pr_init(n, L, psi.ctypes.data, b.ctypes.data, R, alpha, beta0, 0, 0, ctypes.byref(h))

    assert init(100, 0, 5) == -1          # L < 1
    assert init(100, 12, 0) == -1         # R < 1
    assert init(100, 12, 5, alpha=0.0) == -1
    assert init(100, 12, 5, beta0=-1.0) == -1
    assert init(7 * 11, 2, 3) == -8       # prime factors outside {2, 3, 5}
    assert init(2 * 4099, 2, 3) == -8     # 4099 is prime
    rng = np.random.default_rng(0)
    psi = rng.standard_normal((2, 300)) + 1j * rng.standard_normal((2, 300))   # > 256 distinct values
    assert init(300, 2, 3, psi=psi) == -8
    assert h.value is None
