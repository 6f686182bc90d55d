"""Pin the synthetic-scene port (paper_2411_17660_b200/scenes.py) to the reference's
providers (providers.py:65-430): committed golden fixture everywhere, and the live
reference module in the build container."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2411_17660_b200 import scenes
from paper_2411_17660_b200.errors import ConfigError, DataError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "scene_line6.npz")


def _line6():
    spec = scenes.SceneSpec(trajectory="line", frames=6, height=24, width=32, seed=3,
                            pixel_noise=0.05, prior_scale_range=(0.8, 1.2),
                            prior_offset_range=(-0.02, 0.02), prior_noise=0.01)
    return scenes.Scene(spec)


def test_against_golden_fixture():
    g = np.load(GOLD)
    sc = _line6()
    assert np.allclose(sc.intr, g["intr"])
    for k in range(6):
        assert np.allclose(sc.w2c[k][4:], g["w2c"][k][4:], atol=1e-12)
        assert abs(abs(float(sc.w2c[k][:4] @ g["w2c"][k][:4])) - 1.0) < 1e-12
        assert np.allclose(sc.disparity(k), g["disparity"][k], rtol=1e-12)
        assert np.allclose(sc.depth_prior(k), g["prior"][k], rtol=1e-12)
    for e, (i, j) in enumerate(zip(g["ii"], g["jj"])):
        rec = sc.flow_record(int(i), int(j))
        assert np.array_equal(rec[..., 2:], g["flow"][e][..., 2:])  # weights bit-exact
        assert np.abs(rec[..., :2] - g["flow"][e][..., :2]).max() <= 1e-5


def test_against_reference_module(reference_flowsplat):
    _, providers = reference_flowsplat
    for traj in ("orbit", "line", "rotate"):
        spec = providers.SceneSpec(trajectory=traj, frames=10, height=16, width=20, seed=1)
        ref = providers.SyntheticProviders(providers.SyntheticScene(spec))
        mine = scenes.Scene(scenes.SceneSpec(trajectory=traj, frames=10, height=16, width=20, seed=1))
        for i, j in ((0, 1), (4, 6), (9, 7)):
            u = ref.provide_correspondences(i, j)
            t, w = mine.correspondences(i, j)
            assert np.all(np.abs(u.target - t) <= 1e-9 * np.maximum(1.0, np.abs(u.target)))
            assert np.array_equal(u.weight, w)


def test_determinism_and_truth_energy():
    a = _line6().flow_record(2, 3)
    b = _line6().flow_record(2, 3)
    assert a.tobytes() == b.tobytes()


def test_radius_edges_lexicographic():
    ii, jj = scenes.radius_edges(5, 2)
    pairs = list(zip(ii.tolist(), jj.tolist()))
    assert pairs == sorted(pairs)
    assert len(pairs) == 2 * (4 + 3)
    assert all(0 < abs(i - j) <= 2 for i, j in pairs)


def test_configs_shapes():
    wl = scenes.make_workload("C1", height=16, width=24)
    assert wl.flow.shape == (26, 16, 24, 4) and wl.flow.dtype == np.float32
    assert wl.poses0.shape == (8, 7) and wl.fixed.sum() == 1
    assert np.array_equal(wl.poses0[0], wl.true_poses[0])


def test_spec_validation():
    with pytest.raises(ConfigError):
        scenes.SceneSpec(frames=1)
    with pytest.raises(ConfigError):
        scenes.SceneSpec(trajectory="spiral")


def test_dspt_roundtrip(tmp_path):
    arr = np.random.default_rng(0).normal(size=(6, 7, 4)).astype(np.float32)
    p = tmp_path / "flow_000001_000002.dspt"
    scenes.write_dspt(p, arr)
    assert p.stat().st_size == 20 + arr.nbytes
    assert np.array_equal(scenes.read_dspt_f32(p), arr)
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(DataError):
        scenes.read_dspt_f32(p)


def test_workload_mean_flow_distance_matches_graph_oracle():
    """scenes.mean_flow_distance (host numpy, used to build C2's proximity edges) restates G1
    like oracle/graph.py (the bit-exact reference of the GPU graph kernels)."""
    import numpy as np
    from oracle import graph as OG
    from paper_2411_17660_b200 import scenes
    wl = scenes.make_workload("C2", height=24, width=32, keyframes=8)
    for a, b in [(0, 1), (2, 6), (7, 3)]:
        got = scenes.mean_flow_distance(wl.poses0[a], wl.poses0[b], wl.disps0[a], wl.intr0)
        ref = OG.mean_flow_distance(wl.poses0[a], wl.poses0[b], wl.disps0[a], wl.intr0)
        assert abs(got - ref) <= 1e-12 * abs(ref), (a, b, got, ref)


def test_c2_is_a_150_edge_proximity_window():
    """BASELINE configs[1]: 25 keyframes, ~150 proximity edges -- the G3 window pairs (radius
    3, 138 edges) plus the 6 closest farther pairs in both directions."""
    from paper_2411_17660_b200 import scenes
    wl = scenes.make_workload("C2")
    assert len(wl.frames) == 25 and len(wl.ii) == 150
    far = [(int(a), int(b)) for a, b in zip(wl.ii, wl.jj) if abs(int(a) - int(b)) > 3]
    assert len(far) == 12 and all((b, a) in far for a, b in far)
