"""The hinge angle's atan2 (csrc/cr_atan2.cuh), host build on CPU.

The reference computes the hinge angle with std::atan2 (proj/src/elements.cpp:116),
glibc's atan2, which is accurate to about half an ulp but not correctly
rounded. The library evaluates a correctly rounded atan2 instead. Checked
here: correct rounding against mpmath at 200 bits, exact special values, and
the agreement with glibc (math.atan2) on near-flat hinge inputs, where every
disagreement is one ulp at a near-midpoint value. The device build is
compared bitwise with this host build in tests/test_gpu_assembly.py."""
import ctypes
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2008_00409_b200", "libweft_gpu.so")


@pytest.fixture(scope="module")
def cr_atan2():
    lib = ctypes.CDLL(LIB)
    f = lib.weft_hinge_atan2_host
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]

    def run(y, x):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(y)
        assert f(len(y), y.ctypes.data, x.ctypes.data, out.ctypes.data) == 0
        return out
    return run


def families(rng, n):
    """(y, x) draws: the whole plane, near-flat hinges (s << c, the cloth's
    case), folded hinges (c < 0), and wide exponent ranges."""
    u = lambda: rng.uniform(-1, 1, n)
    flat_x = np.abs(u()) * 1e-4 + 1e-6
    yield "plane", u(), u()
    yield "flat", flat_x * u() * 1e-2, flat_x
    yield "folded", u() * 1e-3, -(np.abs(u()) + 1e-3)
    yield "wide", u() * np.exp2(rng.integers(-60, 60, n)), u() * np.exp2(rng.integers(-60, 60, n))


def test_correctly_rounded_vs_mpmath(cr_atan2):
    mp = pytest.importorskip("mpmath")
    mp.mp.prec = 200
    rng = np.random.default_rng(11)
    for name, y, x in families(rng, 600):
        got = cr_atan2(y, x)
        for a, b, g in zip(y, x, got):
            want = float(mp.atan2(mp.mpf(float(a)), mp.mpf(float(b))))
            assert g == want, f"{name}: atan2({a.hex()}, {b.hex()}) = {g.hex()}, correctly rounded {want.hex()}"


def test_special_values_match_libm(cr_atan2):
    z, inf, nan = 0.0, math.inf, math.nan
    pairs = [(z, 1.0), (-z, 1.0), (z, -1.0), (-z, -1.0), (1.0, z), (-1.0, z), (1.0, -z), (z, z), (-z, -z),
             (inf, 1.0), (1.0, inf), (1.0, -inf), (inf, inf), (-inf, -inf), (2.5, 2.5), (-2.5, 2.5),
             (1e-300, 1e300), (1e300, 1e-300), (5e-324, 1.0)]
    y = np.array([p[0] for p in pairs])
    x = np.array([p[1] for p in pairs])
    got = cr_atan2(y, x)
    for a, b, g in zip(y, x, got):
        want = math.atan2(a, b)
        assert np.float64(g).tobytes() == np.float64(want).tobytes(), (a, b, g, want)
    got = cr_atan2(np.array([nan, 1.0]), np.array([1.0, nan]))
    assert np.isnan(got).all()


def test_agreement_with_glibc(cr_atan2):
    """Every disagreement with glibc is one ulp; near-flat hinges (the cloth's
    inputs) disagree rarely."""
    rng = np.random.default_rng(3)
    rates = {}
    for name, y, x in families(rng, 200_000):
        got = cr_atan2(y, x)
        ref = np.array([math.atan2(a, b) for a, b in zip(y.tolist(), x.tolist())])
        diff = got != ref
        if diff.any():
            ulps = np.abs(got[diff].view(np.int64) - ref[diff].view(np.int64))
            assert ulps.max() == 1, name
        rates[name] = diff.mean()
    assert rates["flat"] < 1e-4 and rates["folded"] < 1e-4, rates
    assert max(rates.values()) < 2e-3, rates
