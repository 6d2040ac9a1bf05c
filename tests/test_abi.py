"""C-ABI boundary checks that need no GPU: the in-tree library loads,
exports every entry point include/seghull_b200.h declares, and its host
self-test of the glibc-hypot port (used on the device for eps and 2D edge
thresholds) is bit-identical to np.hypot."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1201_2936_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = []
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        syms += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(sh_[a-z0-9_]+)\s*\(", txt, flags=re.M)
    return sorted(set(syms))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_version_string():
    assert b"sm_100a" in _lib.lib().sh_version()


def _hypot_host(x, y):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = np.empty_like(x)
    _lib.lib().sh_hypot_host(x.ctypes.data, y.ctypes.data, out.ctypes.data, x.size)
    return out


def test_glibc_hypot_port_bit_exact():
    rng = np.random.default_rng(0)
    n = 2_000_000
    # wide-range and edge-like (differences of unit-box coordinates) inputs
    a = rng.standard_normal(n) * np.exp2(rng.integers(-600, 600, n))
    b = rng.standard_normal(n) * np.exp2(rng.integers(-600, 600, n))
    c = rng.random(n) - rng.random(n)
    d = rng.random(n) - rng.random(n)
    for x, y in ((a, b), (c, d), (c, c * 1e-9), (a, a)):
        assert _hypot_host(x, y).tobytes() == np.hypot(x, y).tobytes()
    sp = np.array([0.0, -0.0, 1e-320, 5e-324, 1e308, np.inf, -np.inf])
    X, Y = np.meshgrid(sp, sp)
    assert _hypot_host(X.ravel(), Y.ravel()).tobytes() == np.hypot(X.ravel(), Y.ravel()).tobytes()


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = _lib.lib().sh_create(0, ctypes.byref(h))
    assert rc != _lib.SH_OK
    assert _lib.last_error()


def test_workspace_bytes_host_side():
    L = _lib.lib()
    assert L.sh_workspace_bytes(4, 10) == -1 and L.sh_workspace_bytes(2, 0) == -1
    b2 = L.sh_workspace_bytes(2, 100_000_000)
    b3 = L.sh_workspace_bytes(3, 10_000_000)
    # ping-pong record streams (2 buffers x K streams x (8 dim + 4) B, n plus
    # 1/16 + round-1 slack for DEAD padding) plus segment tables sized n / 8
    # (C2: 8.6 GB + 2.4 GB + cursors/keys)
    assert 2 * 2 * 20 * 100_000_000 <= b2 <= 1.6 * 2 * 2 * 20 * 100_000_000
    assert 2 * 3 * 28 * 10_000_000 <= b3 <= 1.6 * 2 * 3 * 28 * 10_000_000
    assert L.sh_workspace_bytes(2, 2_000_000) < b2
