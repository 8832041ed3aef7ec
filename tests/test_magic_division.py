"""The kernel divides by launch-invariant integers (the split count s, the tiles per page) with
m = ceil(2^38 / d) and floor(x / d) = (x m) >> 38 (csrc/internal.h div_magic).  The claim: exact
whenever x d < 2^38.  Checked here by brute force on the ranges the kernel uses: x < 2^25 split
units with s <= 256, products i r < 2^16, and tile indices < 2^25 with tiles per page < 2^13."""

import random


def magic(d):
    return ((1 << 38) + d - 1) // d


def div(x, d):
    return (x * magic(d)) >> 38


def test_exact_on_kernel_ranges():
    rng = random.Random(7)
    for d in range(1, 257):                       # split counts (MAX_FORCED_SPLITS = 256)
        xs = list(range(0, 4096)) + [(1 << 25) - 1, (1 << 16) - 1]
        xs += [k * d + d - 1 for k in ((1 << 25) // d - 1, (1 << 16) // d - 1)]   # worst remainders
        xs += [rng.randrange(1 << 25) for _ in range(2000)]
        for x in xs:
            assert div(x, d) == x // d, (x, d)
    for d in (1, 2, 3, 5, 7, 1000, 4095, 4096, 8191):   # tiles per page (page_size <= 2^18)
        for x in [rng.randrange(1 << 25) for _ in range(5000)] + [(1 << 25) - 1]:
            assert div(x, d) == x // d, (x, d)


def test_bound_is_needed():
    # the exactness condition is not vacuous: past x d < 2^38 the shortcut can fail
    d = 3                                         # m d = 2^38 + 2: the overshoot is 2 x / (3 2^38)
    x = next(x for x in range(1 << 37, (1 << 37) + 10) if div(x, d) != x // d)
    assert x % d == d - 1 and x * d >= 1 << 38
