"""Exact number formatting used by the GPU timeline writer (csrc/numfmt.cuh),
checked on the host against CPython's float repr / json.dumps / int().

The timeline JSON of the reference is json.dump of Python floats and ints
(sinks.py:374-375, :407, :417); the formatter must reproduce those bytes."""

import ctypes as C
import json
import math
import random
import struct
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def nf(tmp_path_factory):
    out = tmp_path_factory.mktemp("nf") / "libnf.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-std=c++17", str(HERE / "native" / "numfmt_host.cpp"),
                    "-o", str(out)], check=True)
    L = C.CDLL(str(out))
    L.nf_double.argtypes = [C.c_double, C.c_char_p]
    L.nf_ns.argtypes = [C.c_int64, C.c_uint64, C.c_char_p]
    L.nf_int_of_double.argtypes = [C.c_double, C.c_char_p]
    L.nf_i128.argtypes = [C.c_int64, C.c_uint64, C.c_char_p]
    return L


def _call(fn, *args):
    buf = C.create_string_buffer(512)
    n = fn(*args, buf)
    return buf.raw[:n].decode()


def _split(n):
    n &= (1 << 128) - 1
    hi = n >> 64
    if hi >= 1 << 63:
        hi -= 1 << 64
    return hi, n & ((1 << 64) - 1)


def _bits(b):
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def test_double_special(nf):
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5, 0.0001234,
            5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 2 ** 53, 2 ** 53 + 2, 2 ** 60,
            123456789.123, 1e22, 1e23, 3.14159, float("inf"), float("-inf"), float("nan"),
            0.3, 2.675, 1.005, 100.0, 1234567890123456.7]
    for v in vals:
        assert _call(nf.nf_double, float(v)) == json.dumps(float(v)), v


def test_double_random_bits(nf):
    rng = random.Random(1234)
    for _ in range(60000):
        v = _bits(rng.getrandbits(64))
        if math.isnan(v):
            continue
        assert _call(nf.nf_double, v) == json.dumps(v), (v, v.hex())


def test_double_random_ranges(nf):
    rng = random.Random(99)
    for _ in range(40000):
        e = rng.randint(-30, 30)
        v = rng.random() * 10.0 ** e * rng.choice((1, -1))
        assert _call(nf.nf_double, v) == json.dumps(v), v
        n = rng.getrandbits(rng.randint(1, 70))
        v = float(n)
        assert _call(nf.nf_double, v) == json.dumps(v), v


def test_ns_div1000(nf):
    rng = random.Random(7)
    cases = [0, 1, -1, 999, 1000, 1001, 123456789, -123456789, 2 ** 53 - 1, 2 ** 53, 2 ** 53 + 1,
             8796093022207999, 8796093022208000, 8796093022208001, 2 ** 63 - 1, -(2 ** 63), 2 ** 64 - 1,
             2 ** 64 + 12345, -(2 ** 64) - 7, 2 ** 100 + 3]
    for _ in range(40000):
        cases.append(rng.getrandbits(rng.randint(1, 66)) * rng.choice((1, -1)))
    for n in cases:
        hi, lo = _split(n)
        assert _call(nf.nf_ns, hi, lo) == json.dumps(n / 1000.0), n


def test_int_of_double(nf):
    rng = random.Random(5)
    vals = [0.0, -0.0, 0.9, -0.9, 1.5, -1.5, 2.0 ** 63, -(2.0 ** 64), 1e300, -1.7976931348623157e308, 12345.678]
    for _ in range(20000):
        v = _bits(rng.getrandbits(64))
        if math.isfinite(v):
            vals.append(v)
    for v in vals:
        assert _call(nf.nf_int_of_double, v) == str(int(v)), v


def test_i128(nf):
    rng = random.Random(3)
    vals = [0, 1, -1, 2 ** 64, 2 ** 64 - 1, -(2 ** 64), 2 ** 127 - 1, -(2 ** 127), 10 ** 20, -(10 ** 25)]
    vals += [rng.getrandbits(rng.randint(1, 127)) * rng.choice((1, -1)) for _ in range(20000)]
    for v in vals:
        hi, lo = _split(v)
        assert _call(nf.nf_i128, hi, lo) == str(v), v
