"""The C-ABI library builds, loads without a GPU and exports every symbol that
include/sylv_sketch.h declares; the binding refuses to run without the library.
(No compute calls: this runs on the CPU-only container.)"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "sylv_sketch.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sylv_[a-z_]+)\s*\(", txt)))


def test_build_and_exports():
    from paper_2311_16019_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/sylv_sketch.h but not exported"


def test_binding_loads_and_reports_version():
    import paper_2311_16019_b200 as pkg
    pkg.load_library()
    assert "sm_100a" in pkg.version()
    assert set(pkg.SYMBOLS) <= set(_declared())


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2311_16019_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_config_is_rejected_without_gpu_work():
    """Argument validation happens before any device call."""
    import numpy as np
    import paper_2311_16019_b200 as pkg
    A = pkg.stencil_operator("stencil2d", 8, (1.0, 1.0))
    C = np.zeros((64, 3))
    with pytest.raises(pkg.SylvError) as e:
        pkg.SylvSketch(A, A, C, C, r=3, k=2, d_max=5, s=64)
    assert e.value.status == 1
    with pytest.raises(pkg.SylvError) as e:
        pkg.SylvSketch(A, A, C[:, :2], C[:, :2], r=2, k=2, d_max=5, s=60)   # s % zeta != 0
    assert e.value.status == 1
