"""The device's host-libm-exact exp and correctly rounded log (csrc/libm_exact.cuh),
built for the host from the same source (tests/native/host_libm_exact.cpp) -- the CPU
half of the check; tests/test_refcdf.py runs the device half on the B200.

The reference's resampling CDF (engine.cpp:61-80) is a chain of std::exp calls; glibc's
exp is what the reference runs, so the device restates it (ARM optimized-routines
algorithm, x86-64 FMA build).  Pinned here against the host libm bit for bit."""
import ctypes as C
import math
import os
import subprocess
from decimal import Decimal, getcontext

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2408_12057_b200", "csrc")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("libm") / "host_libm_exact.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "native", "host_libm_exact.cpp"), "-o", str(out), "-lm"],
                   check=True)
    L = C.CDLL(str(out))
    for f in ("host_gexp", "host_crlog"):
        getattr(L, f).argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_double)]
    L.host_sweep.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    return L


def call(L, f, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    getattr(L, f)(x.ctypes.data_as(C.POINTER(C.c_double)), len(x), out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def test_table_generator_matches_header():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "tools", "gen_exp_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    src = open(os.path.join(CSRC, "libm_exact.cuh")).read()
    body = src[src.index("kExpTab[256] = {"):src.index("};", src.index("kExpTab[256] = {"))]
    words = [int(w, 16) for w in body.replace("ull", "").replace(",", " ").split()[3:] if w.startswith("0x")]
    assert words == [v for pair in gen.table() for v in pair]


def test_gexp_equals_host_libm_bit_for_bit(lib):
    eb, lb = C.c_uint64(), C.c_uint64()
    lib.host_sweep(4_000_000, 0x9E3779B97F4A7C15, C.byref(eb), C.byref(lb))
    assert eb.value == 0
    # special arguments
    h = float.fromhex
    xs = np.array([0.0, -0.0, 1e-300, -1e-300, h('0x1p-54'), -h('0x1p-54'), -745.13321910194122, -745.2, -746.0,
                   -708.39641853226408, 709.78271289338397, 709.8, -np.inf, np.inf, -1022 * math.log(2),
                   -1074 * math.log(2), 512.0, -512.0, 1023.9, -1e9])
    got = call(lib, "host_gexp", xs)
    ref = np.array([math.exp(x) if x < 709.8 else float("inf") for x in xs])
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_crlog_is_correctly_rounded_and_near_glibc(lib):
    getcontext().prec = 60
    g = np.random.default_rng(3)
    ys = np.concatenate([1.0 + g.random(3000) * 4194303.0, g.random(500) * 4 + 1e-3,
                         [1.0, 2.0, 0.5, 1 + 2**-52, 3.0, 2**-1074, 1e308]])
    got = call(lib, "host_crlog", ys)
    for y, v in zip(ys, got):
        exact = Decimal(float(y)).ln()
        assert v == float(exact), (y, v, float(exact))
    eb, lb = C.c_uint64(), C.c_uint64()
    n = 2_000_000
    lib.host_sweep(n, 12345, C.byref(eb), C.byref(lb))
    # glibc's log is a 0.52-ulp algorithm: it misrounds a small fraction of arguments
    assert lb.value / n < 2e-3, lb.value / n
