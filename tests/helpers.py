"""Shared test helpers: tolerances and comparisons."""

import numpy as np

# north_star: max-abs 2e-3 and max-rel 1e-2 for bf16 inputs with fp32 accumulation, read as
# an allclose bound per element (C-amb-14); lse within 1e-4 absolute.
OUT_ATOL = 2e-3
OUT_RTOL = 1e-2
LSE_ATOL = 1e-4


def assert_out_close(got, ref, what="out"):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    err = np.abs(got - ref)
    bound = OUT_ATOL + OUT_RTOL * np.abs(ref)
    bad = err > bound
    if bad.any():
        idx = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} elements out of tolerance; worst at {idx}: "
                             f"got {got[idx]!r} ref {ref[idx]!r} (max abs err {err.max():.3g})")


def assert_lse_close(got, ref, what="lse"):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape
    ninf_ref = np.isneginf(ref)
    assert (np.isneginf(got) == ninf_ref).all(), f"{what}: -inf pattern differs"
    fin = ~ninf_ref
    if fin.any():
        err = np.abs(got[fin] - ref[fin])
        assert err.max() <= LSE_ATOL, f"{what}: max abs err {err.max():.3g} > {LSE_ATOL}"
