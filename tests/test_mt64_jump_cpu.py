"""mt19937_64 jump-ahead, host half (no GPU): the product's jump
polynomials (mg_mt64_jump_polynomial: Berlekamp-Massey characteristic
polynomial + square-and-multiply, paper_2309_15676_b200/csrc/mt64_jump.cu)
applied by the oracle's bit-by-bit Horner restatement reproduce the
sequential stream exactly: jump(J) == discard(J)."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    L.mg_mt64_jump_polynomial.argtypes = [C.c_uint64, C.c_void_p, C.POINTER(C.c_int32)]
    return L


def poly(lib, J):
    w = np.zeros(312, dtype=np.uint64)
    deg = C.c_int32()
    assert lib.mg_mt64_jump_polynomial(J, w.ctypes.data_as(C.c_void_p), C.byref(deg)) == 0
    return w, deg.value


@pytest.mark.parametrize("J", [1, 2, 311, 312, 313, 1000, 4096 * 3 - 7, 123457])
def test_jump_equals_discard(lib, oracle, J):
    w, deg = poly(lib, J)
    L = oracle.lib
    L.mgo_mt64_jump.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.mgo_mt64_next.restype = C.c_uint64
    L.mgo_mt64_next.argtypes = [C.c_void_p]
    g = oracle.new_stream(42, 7)
    L.mgo_mt64_jump(g, w.ctypes.data_as(C.c_void_p), deg)
    jumped = [L.mgo_mt64_next(g) for _ in range(700)]
    seq = oracle.rng_draws(42, 7, 1, J + 700)[J:]
    assert np.array_equal(np.array(jumped, dtype=np.uint64), seq)


def test_jump_polynomial_identities(lib):
    # x^1 mod phi = x ; x^0 = 1 ; degrees stay below 19937
    w, deg = poly(lib, 1)
    assert deg == 1 and w[0] == 2 and not w[1:].any()
    w, deg = poly(lib, 19936)
    assert deg == 19936
    w, deg = poly(lib, 10 ** 12)
    assert 0 <= deg < 19937
