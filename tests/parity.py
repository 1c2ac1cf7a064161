"""Element-by-element parity bounds shared by the GPU tests.

The north star's gate is normwise (‖gpu − ref‖₂/‖ref‖₂ ≤ 2e-2 for bf16,
reading R14), which a handful of wrong elements in a large tensor can pass.
Every GPU parity test therefore also bounds EACH element:

    |gpu − ref| ≤ ulps · ulp_bf16(ref) + atol_rms · rms(ref)

ulp_bf16(x) is the bf16 spacing at |x| (2^(e−8) for |x| ∈ [2^(e−1), 2^e)):
both sides round the same real value to bf16, so a correct kernel differs
from the oracle by at most one rounding step, plus an absolute term for
elements near zero whose accumulation order differs (fp32 sums, the bf16
probabilities of attention, chained kernels). A wrong element (bad index,
dropped term, stale landing slot) is off by O(rms) and fails.
"""
import numpy as np


def bf16_ulp(x):
    x = np.abs(np.asarray(x, np.float64))
    _, e = np.frexp(x)
    return np.where(x > 0, np.ldexp(1.0, e - 8), 0.0)


def assert_elementwise(got, ref, ulps=1.0, atol_rms=1e-3, what="output"):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    assert np.all(np.isfinite(got)), f"{what}: non-finite values"
    rms = float(np.sqrt(np.mean(ref * ref))) if ref.size else 0.0
    bound = ulps * bf16_ulp(ref) + atol_rms * rms
    err = np.abs(got - ref)
    bad = err > bound
    if bad.any():
        i = np.unravel_index(int(np.argmax(np.where(bad, err - bound, -np.inf))), ref.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} of {ref.size} elements outside {ulps} ulp + "
                             f"{atol_rms}·rms (rms {rms:.3e}); worst at {i}: got {got[i]!r} ref {ref[i]!r}")
    return float(np.max(err / np.maximum(bound, 1e-300))) if ref.size else 0.0
