"""Compact per-iteration disparity fixtures (test infrastructure).

A float32 (N,H,W) disparity map per GN iteration of the 300-frame C3 config is 3.7 MB;
eight of them, for the clean and the noisy variant, would put ~60 MB of incompressible
mantissas into git.  The parity bar is 1e-4 relative, so the fixtures store
q = round(log(d) / QUANT) as int32 -- 5e-7 relative at worst, 200x below the bar -- as
differences from the previous iteration (iteration 0 = the workload's own input
disparities, recomputed at load time), which zlib packs tightly once the solve has
converged.
"""

from __future__ import annotations

import numpy as np

QUANT = 1e-6


def quantize(d) -> np.ndarray:
    return np.rint(np.log(np.asarray(d, np.float64)) / QUANT).astype(np.int64)


def encode(d0, disps):
    """d0 (N,H,W) input, disps: list of (N,H,W) per iteration -> list of int32 deltas."""
    prev = quantize(d0)
    out = []
    for d in disps:
        q = quantize(d)
        delta = q - prev
        if np.abs(delta).max() >= 2**31:
            raise ValueError("disparity change too large for the int32 codec")
        out.append(delta.astype(np.int32))
        prev = q
    return out


def decode(d0, deltas):
    """Inverse of ``encode``: list of float64 (N,H,W) disparities per iteration."""
    q = quantize(d0)
    out = []
    for dl in deltas:
        q = q + dl.astype(np.int64)
        out.append(np.exp(q * QUANT))
    return out
