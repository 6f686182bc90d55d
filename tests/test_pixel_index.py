"""The kernels map a flat pixel index p to (u, v) without integer division:
v = floor((p + 0.5) * (1/W)), u = fma(-v, W, p) in float64 (dba_pass.cuh / dba_energy.cuh).
IEEE float64 multiply and floor behave the same on the host, so the exactness claim (every
p < 2^40 for any realistic W) is checked here against integer division."""

import numpy as np
import pytest


@pytest.mark.parametrize("W", [1, 3, 7, 16, 31, 64, 100, 333, 640, 1023, 1920, 4096, 7681])
def test_floor_row_index_is_exact(W):
    rng = np.random.default_rng(W)
    H = 4096
    p = np.concatenate([np.arange(0, min(W * H, 1 << 16), dtype=np.int64),
                        rng.integers(0, W * H, size=1 << 16, dtype=np.int64),
                        np.arange(W - 2, W * H, W, dtype=np.int64),  # row ends and starts
                        np.arange(W, W * H, W, dtype=np.int64)])
    p = p[(p >= 0) & (p < W * H)]
    pd = p.astype(np.float64)
    iW = 1.0 / float(W)
    v = np.floor((pd + 0.5) * iW)
    u = pd - v * float(W)  # exact: v * W and the difference are integers below 2^53
    assert np.array_equal(v.astype(np.int64), p // W)
    assert np.array_equal(u.astype(np.int64), p % W)
