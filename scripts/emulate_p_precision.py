"""CPU emulation of the PV product's precision: P = exp(S - m) rounded to ONE bf16 (FA-style)
versus the unevaluated bf16 pair P_hi + P_lo the kernel uses (csrc/fwd.cu mma_tile), against the
exact fp64 result, as max over rows of |err| / (2e-3 + 1e-2 |ref|) (C-amb-14's per-element bound;
> 1 fails).  G = 8 query rows, d = 128, q/K/V ~ N(0,1) bf16 (peak = 8 scales q: the "peaked"
variant).  Output: profiles/r01g_p_precision.txt.
"""
import numpy as np, torch
def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float32).numpy().astype(np.float64)
rng = np.random.default_rng(0)
def trial(n, peak, hilo, G=8, d=128):
    q = bf16(rng.standard_normal((G, d)) * peak); k = bf16(rng.standard_normal((n, d))); v = bf16(rng.standard_normal((n, d)))
    s = (q @ k.T) / np.sqrt(d)
    m = s.max(1, keepdims=True)
    p = np.exp(s - m)
    ref = (p @ v) / p.sum(1, keepdims=True)
    p32 = p.astype(np.float32)
    ph = bf16(p32)
    if hilo:
        pl = bf16(p32 - ph.astype(np.float32)); pe = ph + pl
    else:
        pe = ph
    out = (pe @ v) / p32.astype(np.float64).sum(1, keepdims=True)
    out = bf16(out)
    ratio = np.abs(out - ref) / (2e-3 + 1e-2 * np.abs(ref))
    return ratio.max()
for peak in (1, 8):
    for n in (1, 2, 3, 4, 6, 8, 16, 32, 64, 128, 512):
        r1 = max(trial(n, peak, False) for _ in range(60))
        r2 = max(trial(n, peak, True) for _ in range(60))
        print(f"peak={peak} n={n:4d}: max err/bound single-bf16 {r1:.3f}   hi/lo {r2:.3f}")
