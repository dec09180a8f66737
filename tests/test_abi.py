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


@pytest.mark.parametrize("kind,N,n", [("stencil3d", 256, 256 ** 3), ("stencil2d", 512, 512 * 512),
                                      ("csr", 1, 4194304), ("csr", 1, 20011)])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_tiles_rows_on_32_row_groups(kind, N, n, P):
    """sylv_partition (host only): the ranks' ranges tile [0, n) in order, start at multiples
    of 32 rows (the sketch hash's groups never straddle ranks), are whole planes / lines for
    the stencils, and are balanced to within one plane group / one 32-row group."""
    import paper_2311_16019_b200 as pkg
    from synth import inputs
    cfg = inputs.small_config(kind=kind, N=N, n=n) if kind == "csr" else inputs.small_config(kind=kind, N=N)
    rows = [pkg.partition(cfg, P, r) for r in range(P)]
    assert rows[0][0] == 0 and rows[-1][1] == cfg.n
    assert all(rows[i][1] == rows[i + 1][0] for i in range(P - 1))
    assert all(b % 32 == 0 and e > b for b, e in rows)
    unit = N * N if kind == "stencil3d" else N if kind == "stencil2d" else 1
    assert all(b % unit == 0 and (e % unit == 0 or e == cfg.n) for b, e in rows)
    sizes = [e - b for b, e in rows]
    g = 32 if kind == "csr" else max(unit, 32)
    assert max(sizes) - min(sizes) <= 2 * g


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the oracle arm, CPU only) prints one JSON line with the
    contract's keys (c0, a few steps)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "c0",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_buffer_checks_refuse_wrong_dtype_shape_and_copies():
    """The binding passes raw double* to the library: a wrong dtype, a wrong shape or a
    non-contiguous numpy output (which would be silently copied and the result lost) must be
    refused before the C call."""
    import numpy as np
    from paper_2311_16019_b200.api import _ptr
    good = np.zeros((10, 4))
    assert _ptr(good, shape=(10, 4), out=True)[0] == good.ctypes.data
    with pytest.raises(ValueError):
        _ptr(np.zeros((10, 4), dtype=np.float32), shape=(10, 4), out=True)
    with pytest.raises(ValueError):
        _ptr(np.zeros((10, 3)), shape=(10, 4), out=True)
    with pytest.raises(ValueError):
        _ptr(np.zeros((4, 10)).T, shape=(10, 4), out=True)          # non-contiguous output
    with pytest.raises(ValueError):
        _ptr(np.zeros((9, 4)), shape=(10, 4))                       # input of the wrong shape
    p, keep = _ptr(np.zeros((4, 10)).T, shape=(10, 4))              # inputs may be copied
    assert keep.flags.c_contiguous and keep.shape == (10, 4)
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError):
        _ptr(torch.zeros((10, 4), dtype=torch.float32), shape=(10, 4))
    with pytest.raises(ValueError):
        _ptr(torch.zeros((4, 10), dtype=torch.float64).t(), shape=(10, 4))


def test_config_struct_layout_matches_header():
    """sylv_config fields in the ctypes mirror appear in the header in the same order (the
    struct is passed by pointer: a missing or reordered field corrupts every later one)."""
    from paper_2311_16019_b200.api import Config
    txt = open(os.path.join(ROOT, "include", "sylv_sketch.h")).read()
    body = txt[txt.index("typedef struct {\n  int32_t r;"):txt.index("} sylv_config;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b([a-z_0-9]+)\s*;", body)
    assert fields == [f for f, _ in Config._fields_]
