"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/wave.h declares, validates descriptors, sizes buffers, decomposes the
domain (SPEC.md L239-247 examples) and builds constants that agree bitwise
with the independently written oracle (both: fp64 compute, one fp32 rounding)."""
import json
import os
import re

import numpy as np
import pytest

from paper_2009_04619_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build_cuda()
    return _abi.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "wave.h")).read()
    return sorted(set(re.findall(r"WAVE_API[^;(]*?\b(wave_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_abi.EXPORTS) == syms


def test_version(L):
    assert "sm_100a" in _abi.wave_version()


def test_layout():
    d = _abi.make_desc(70, 45, 53, 5, 7.5, 6e-4)
    lay = _abi.wave_layout(d)
    assert lay.pitch_x == 72 and lay.pitch_x % 4 == 0
    assert lay.ghost_z == 4 and lay.planes == 61
    assert lay.elems_u == 61 * 45 * 72 and lay.elems_vdt2 == 53 * 45 * 72
    assert lay.align_bytes == 128


@pytest.mark.parametrize("kw,msg", [
    (dict(nx=0), "extents"),
    (dict(pml_width=32), "2w"),
    (dict(h=0.0), "spacing"),
    (dict(dt=-1.0), "dt"),
    (dict(eta_max=-1.0), "eta_max"),
    (dict(nz=40, nz_global=64, z_offset=30), "slab"),
    (dict(kernel=7), "kernel"),
    (dict(dt=0.0, nz=32, nz_global=64), "auto dt"),
])
def test_validation_errors(L, kw, msg):
    base = dict(nx=64, ny=64, nz=64, pml_width=16, h=10.0, dt=2e-3, eta_max=4.0)
    base.update(kw)
    with pytest.raises(_abi.WaveError) as e:
        _abi.wave_layout(_abi.make_desc(**base))
    assert e.value.status == _abi.WAVE_ERR_CONFIG
    assert msg in e.value.message


def test_decompose_golden_12_w2():
    g = GOLD["decompose_12_w2"]
    n = g["extent"]
    regs = _abi.wave_decompose(_abi.make_desc(n, n, n, g["w"], 1.0, 1e-3))
    vols = {r["kind"]: int(np.prod(r["ext"])) for r in regs}
    assert vols == g["volumes"]
    inner = regs[0]
    assert inner["lo"] == (2, 2, 2) and inner["ext"] == (8, 8, 8)


def _membership(nx, ny, nz, w):
    regs = _abi.wave_decompose(_abi.make_desc(nx, ny, nz, w, 1.0, 1e-3))
    cnt = np.zeros((nz, ny, nx), np.int32)
    for r in regs:
        (x, y, z), (ex, ey, ez) = r["lo"], r["ext"]
        assert min(ex, ey, ez) >= 0
        cnt[z:z + ez, y:y + ey, x:x + ex] += 1
    return cnt, regs


def test_decompose_partition_examples():
    g = GOLD["decompose_16x12x10_w2"]
    cnt, regs = _membership(*g["extents"], g["w"])
    assert (cnt == 1).all() and cnt.sum() == g["total"]
    cnt, regs = _membership(9, 9, 9, 0)          # w = 0: inner is everything
    assert (cnt == 1).all() and regs[0]["ext"] == (9, 9, 9)


def test_decompose_partition_random():
    rng = np.random.default_rng(0)
    for _ in range(200):
        nx, ny, nz = (int(v) for v in rng.integers(1, 24, 3))
        wmax = (min(nx, ny, nz) - 1) // 2
        w = int(rng.integers(0, wmax + 1))
        cnt, _ = _membership(nx, ny, nz, w)
        assert (cnt == 1).all(), (nx, ny, nz, w)


@pytest.mark.parametrize("h,dt,eta,w", [
    ((10.0, 10.0, 10.0), 2e-3, 4.0, 16),
    ((7.5, 7.5, 7.5), 6e-4, 4.0, 5),
    ((10.0, 8.0, 12.5), 8.888889e-4, 30.0, 3),
    ((1.0, 2.0, 4.0), 1e-3, 0.0, 0),
])
def test_constants_match_oracle_bitwise(L, oracle_lib, h, dt, eta, w):
    import oracle
    d = _abi.make_desc(64, 64, 64, w, h, float(np.float32(dt)), eta)
    a = _abi.wave_constants(d)
    b = oracle.constants(oracle.make_geom(64, 64, 64, w, h, dt, eta), round32=True, dtype=np.float32)
    for k in ("c_x", "c_y", "c_z", "eta", "A", "B", "inv2h"):
        assert np.array_equal(a[k], b[k]), k
    assert a["c_xyz"] == b["c_xyz"]


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    # the product path must fail loudly without the CUDA library
    monkeypatch.setattr(_abi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(ImportError):
        _abi.lib()


def test_layout_fp64_element_size():
    d32 = _abi.make_desc(70, 45, 53, 5, 7.5, 6e-4)
    d64 = _abi.make_desc(70, 45, 53, 5, 7.5, 6e-4, precision=_abi.WAVE_PREC_FP64)
    l32, l64 = _abi.wave_layout(d32), _abi.wave_layout(d64)
    assert l32.elem_bytes == 4 and l64.elem_bytes == 8
    # same element counts: the layout is in elements of the plan's precision
    assert (l32.pitch_x, l32.elems_u, l32.elems_vdt2) == (l64.pitch_x, l64.elems_u, l64.elems_vdt2)


@pytest.mark.parametrize("kw,msg", [
    (dict(precision=2), "precision"),
    (dict(precision=_abi.WAVE_PREC_FP64, kernel=_abi.WAVE_KERNEL_TB2), "TB2"),
])
def test_precision_validation(kw, msg):
    d = _abi.make_desc(70, 45, 53, 5, 7.5, 6e-4, **kw)
    with pytest.raises(_abi.WaveError) as ei:
        _abi.wave_layout(d)
    assert ei.value.status == _abi.WAVE_ERR_CONFIG and msg in ei.value.message


def test_host_only_calls_accept_tb2_fp32():
    d = _abi.make_desc(70, 45, 53, 5, 7.5, 6e-4, kernel=_abi.WAVE_KERNEL_TB2)
    assert _abi.wave_layout(d).elems_u == 61 * 45 * 72
