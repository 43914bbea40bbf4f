"""Output tolerances of the parity tests (R28).

fp32 path: max-abs 1e-4 (north_star).  bf16 path: max-abs 2e-2 (north_star) on the compute,
plus, where it exceeds that budget, the output's own RNE rounding (R13): the exact result is
not representable in bf16, and for |o| >= 4 half a bf16 ulp is already 0.0156 of the 0.02.
Element-wise bound: max(2e-2, half_ulp_bf16(|o_ref|) + 1e-2).  Only elements with |o_ref| >= 4
(peaked attention onto a single large v entry: the sharp-q stress inputs) get more than 2e-2.
LSE: max-abs 1e-3 (north_star)."""
import numpy as np

BF16_TOL = 2e-2
F32_TOL = 1e-4
LSE_TOL = 1e-3


def half_ulp_bf16(x):
    """Half the spacing of bf16 values at |x| (8 significant bits)."""
    a = np.abs(np.asarray(x, dtype=np.float64))
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, 2.0 ** (e - 8), 0.0)


def bf16_bound(o_ref):
    return np.maximum(BF16_TOL, half_ulp_bf16(o_ref) + 1e-2)


def out_excess(o, o_ref, bf16: bool):
    """max over elements of |o - o_ref| - bound (<= 0: within tolerance)."""
    err = np.abs(np.asarray(o, dtype=np.float64) - o_ref)
    if err.size == 0:
        return 0.0
    bound = bf16_bound(o_ref) if bf16 else F32_TOL
    return float((err - bound).max())


def assert_out_close(o, o_ref, bf16: bool, what=""):
    err = np.abs(np.asarray(o, dtype=np.float64) - o_ref)
    ex = out_excess(o, o_ref, bf16)
    assert ex <= 0.0, f"{what}: out max-abs {err.max():.3e} exceeds its bound by {ex:.3e}"
    return float(err.max()) if err.size else 0.0
