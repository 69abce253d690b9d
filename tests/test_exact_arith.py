"""The eval kernel's call-free correctly rounded sqrt / division
(vx_internal.cuh: sqrt_rn_nc, div_rn_nc) against the CUDA IEEE intrinsics
__dsqrt_rn / __ddiv_rn, bit for bit, on seeded random inputs spanning the
range Geo::fast_arith admits (squared distances down to 2^-348, growth rates
in [2^-64, 2^64]).  The timed kinds' labels and values depend on these being
exactly the reference's sqrt(d) / G (geometry.hpp:128-135)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("growth", [1.1, 0.9, 3.0, 1.0 / 3.0, 7.25, 0.37, 1e-3, 1e3, 2.0 ** -60, 2.0 ** 60,
                                    0.7, 1.2, 0.5 * (1 + 5 ** 0.5)])
def test_call_free_sqrt_and_division_are_ieee(growth):
    from paper_2201_13234_b200._lib import check, lib

    bs, bd = C.c_uint64(0), C.c_uint64(0)
    check(lib().vx_probe_exact_arith(0, 1 << 27, 0x5eed ^ hash(growth) & 0xFFFFFFFF, growth, C.byref(bs), C.byref(bd)))
    assert bs.value == 0 and bd.value == 0, (bs.value, bd.value)


def test_call_free_division_random_growth():
    from paper_2201_13234_b200._lib import check, lib

    rng = np.random.default_rng(77)
    for g in np.exp2(rng.uniform(-64, 64, 24)):
        bs, bd = C.c_uint64(0), C.c_uint64(0)
        check(lib().vx_probe_exact_arith(0, 1 << 24, int(rng.integers(1 << 62)), float(g), C.byref(bs), C.byref(bd)))
        assert bs.value == 0 and bd.value == 0, (float(g), bs.value, bd.value)
