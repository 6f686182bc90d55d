"""GPU synthetic correspondence provider vs the CPU scene port
(scenes.Scene.flow_record, itself pinned to the reference provider in test_scenes.py)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2411_17660_b200 import scenes


@pytest.mark.gpu
@pytest.mark.parametrize("traj,frames,noise", [("orbit", 300, 0.0), ("line", 100, 0.0), ("orbit", 300, 0.5)])
def test_gpu_flows_match_cpu_provider(traj, frames, noise):
    from paper_2411_17660_b200.provider import synthetic_flows
    sc = scenes.Scene(scenes.SceneSpec(trajectory=traj, frames=frames, height=48, width=64, seed=0,
                                       pixel_noise=noise))
    ii, jj = scenes.radius_edges(8, 3)
    ii, jj = ii * 3, jj * 3  # wider baselines: more occlusion and out-of-view pixels
    got = synthetic_flows(sc, ii, jj).cpu().numpy()
    exp = np.stack([sc.flow_record(int(i), int(j)) for i, j in zip(ii, jj)])
    w_got, w_exp = got[..., 2], exp[..., 2]
    assert np.array_equal(got[..., 2], got[..., 3])
    assert np.mean(w_got != w_exp) < 1e-3  # visibility ties at the 1e-6 / bound thresholds only
    both = (w_got > 0) & (w_exp > 0)
    assert both.mean() > 0.3
    err = np.abs(got[..., :2] - exp[..., :2])[both]
    assert err.max() < (1e-3 if noise == 0 else 1e-3 + 1e-5)
