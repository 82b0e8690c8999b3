"""The parity bars of the tensor-core modes, in one place.

* fp64 / fp32: bit equality with the reference's execute() / its f32 mode.
* fp32x3 (fp32-accurate tensor-core contractions): the reference's own metric,
  max_rel_err (tensor.cc:9-19) <= 1e-5 — the north star's fp32 bar.
* tf32 / bf16: normwise, max|got - ref| / max(1, max|ref|) <= 1e-2 / 3e-2.
  max_rel_err's max(1, |ref|) denominator turns into an absolute error for
  outputs near zero, which no 8- or 11-bit operand rounding can bound (a
  bf16 contraction of K terms carries ~2^-9 * sqrt(K) * |x||y| of noise at
  every output, zero or not), so these modes are held to the normwise bound.
"""
import numpy as np

BARS = {"fp32x3": ("max_rel_err", 1e-5), "tf32": ("normwise", 1e-2), "bf16": ("normwise", 3e-2)}


def max_rel_err(got, want):
    """tensor.cc:9-19."""
    g = np.asarray(got, dtype=np.float64).ravel()
    w = np.asarray(want, dtype=np.float64).ravel()
    return float(np.max(np.abs(g - w) / np.maximum(1.0, np.abs(w)))) if w.size else 0.0


def normwise(got, want):
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    if not w.size:
        return 0.0
    return float(np.max(np.abs(g - w))) / max(1.0, float(np.max(np.abs(w))))


def error(prec, got, want):
    """(metric name, value, bar) of a tensor-core mode against the reference."""
    metric, bar = BARS[prec]
    return metric, (max_rel_err if metric == "max_rel_err" else normwise)(got, want), bar


def within(prec, got, want):
    metric, err, bar = error(prec, got, want)
    return err <= bar
