"""The multiply-shift division the weight-gradient gather relies on
(gemm_tc2.cu `divmagic`: m = ceil(2^(31+l) / d), l = ceil(log2 d);
x / d == (x * m) >> (31 + l) for every 0 <= x < 2^31), restated and checked at
the divisors GoogLeNet / NIN / the test shapes produce and at the edge values
where a too-small multiplier would first fail (multiples of d and their
predecessors near 2^31)."""

import random

import pytest


def divmagic(d):
    l = 0
    while (1 << l) < d:
        l += 1
    s = 31 + l
    return ((1 << s) + d - 1) // d, s


DIVISORS = sorted({1, 2, 3, 7, 8, 16, 32, 49, 64, 112, 196, 784, 3136, 12544, 112 * 128,
                   2 ** 20 - 1, 2 ** 24 + 1, 12345, 65535, 1 << 30})


@pytest.mark.parametrize("d", DIVISORS)
def test_multiply_shift_division_is_exact(d):
    m, s = divmagic(d)
    assert m < (1 << 64) and (((1 << 31) - 1) * m) < (1 << 64)  # fits the device's u64 product
    rng = random.Random(d)
    xs = [0, 1, d - 1, d, d + 1, (1 << 31) - 1, (1 << 31) - 2]
    top = ((1 << 31) - 1) // d
    for q in (1, 2, top - 1, top):
        xs += [q * d - 1, q * d, q * d + d - 1]
    xs += [rng.randrange(0, 1 << 31) for _ in range(2000)]
    for x in xs:
        if 0 <= x < (1 << 31):
            assert (x * m) >> s == x // d, (x, d)
