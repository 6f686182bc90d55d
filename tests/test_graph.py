"""Frame-graph construction: oracle pins (SPEC examples,
closed form) on CPU; native builders vs the oracle on CPU; the GPU distance kernel
bitwise against the oracle."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import graph as OG
from paper_2411_17660_b200 import graph, scenes
from tests.helpers import small_workload


def _quat_axis(axis, ang):
    a = np.asarray(axis, float) / np.linalg.norm(axis)
    return np.concatenate([[np.cos(ang / 2)], np.sin(ang / 2) * a])


# ----------------------------------------------------------------- oracle pins (SPEC examples)

def test_oracle_frontend_spec_examples():
    assert OG.frontend_edges([0, 1, 2], radius=2) == [(0, 1), (0, 2), (1, 0), (1, 2), (2, 0), (2, 1)]
    assert (0, 1) not in OG.frontend_edges([0, 1, 2], radius=2, existing=[(0, 1)], ages=[31])
    assert (0, 1) in OG.frontend_edges([0, 1, 2], radius=2, existing=[(0, 1)], ages=[30])
    assert OG.frontend_edges([7], radius=3) == []


def test_oracle_backend_spec_examples():
    rng = np.random.default_rng(0)
    n = 200
    D = rng.uniform(1, 10, size=(n, n))
    e = OG.backend_edges(list(range(n)), D, loops=[(5, 190)])
    assert (5, 190) in e and len(e) <= 1500
    assert all(min(i, j) >= 50 for i, j in e if (i, j) != (5, 190))
    D2 = rng.uniform(1, 10, size=(100, 100))
    assert len(OG.backend_edges(list(range(100)), D2)) <= 1500


def test_oracle_distance_identity_and_closed_form_rotation():
    H, W = 24, 32
    intr = np.array([30.0, 30.0, 15.5, 11.5])
    disp = np.full((H, W), 0.5)
    eye = np.array([1.0, 0, 0, 0, 0, 0, 0])
    assert OG.mean_flow_distance(eye, eye, disp, intr) == 0.0
    # rotation about the optical axis: every pixel turns about (cx, cy) by theta,
    # |flow| = 2 sin(theta/2) |p - c| for both the full and the rotation-only flow
    th = np.deg2rad(3.0)
    rot = np.concatenate([_quat_axis([0, 0, 1], th), [0, 0, 0]])
    u, v = np.meshgrid(np.arange(W), np.arange(H))
    closed = 2 * np.sin(th / 2) * np.hypot(u - intr[2], v - intr[3]).mean()
    for beta in (0.0, 0.5, 1.0):
        assert abs(OG.mean_flow_distance(eye, rot, disp, intr, beta) - closed) < 1e-9 * closed
    # beta = 1: the mean full-flow magnitude alone (translation included)
    tr = np.array([1.0, 0, 0, 0, 0.1, 0, 0])
    sf, nf, _, _ = OG.flow_terms(eye, tr, disp, intr)
    assert OG.mean_flow_distance(eye, tr, disp, intr, 1.0) == sf / nf


# ----------------------------------------------------------------- native builders vs oracle (CPU)

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_backend_builder_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = [12, 60, 170][seed]
    frames = np.sort(rng.choice(1000, size=n, replace=False))
    D = np.round(rng.uniform(0, 5, size=(n, n)), 1)  # many exact ties
    D[rng.uniform(size=(n, n)) < 0.05] = np.inf
    loops = [(int(frames[0]), int(frames[-1]))] if seed else []
    for window, cap in ((150, 1500), (8, 20), (40, 301)):
        exp = OG.backend_edges(frames, D, window, cap, loops)
        ii, jj = graph.backend_edges(frames, D, window, cap, loops)
        assert list(zip(ii.tolist(), jj.tolist())) == exp


@pytest.mark.parametrize("seed", [0, 1])
def test_frontend_builder_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    window = np.sort(rng.choice(100, size=12, replace=False))
    existing = [(int(a), int(b)) for a, b in rng.choice(100, size=(30, 2))]
    ages = rng.integers(0, 40, size=30)
    for radius in (0, 1, 3):
        exp = OG.frontend_edges(window, radius, existing, ages, 30)
        ii, jj = graph.build_frontend_edges(window, radius, existing, ages, 30)
        assert list(zip(ii.tolist(), jj.tolist())) == exp


# ----------------------------------------------------------------- GPU distance kernel

def _graph_scene():
    wl = small_workload("C2", height=24, width=32, keyframes=14, radius=2)
    disps = wl.disps0.copy()
    disps[3, 0, :5] = 0.0      # non-positive disparity: excluded from the full flow
    disps[4, 1, 2] = -1.0
    return wl, disps


@pytest.mark.gpu
def test_frame_distance_bitwise_vs_oracle():
    wl, disps = _graph_scene()
    n = len(wl.frames)
    A, B = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    m = A != B
    for beta in (0.5, 0.7):
        got = graph.frame_distances(wl.poses0, disps, wl.intr0, A[m], B[m], beta)
        exp = np.array([OG.mean_flow_distance(wl.poses0[a], wl.poses0[b], disps[a], wl.intr0, beta)
                        for a, b in zip(A[m], B[m])])
        assert np.array_equal(got, exp)


@pytest.mark.gpu
def test_backend_graph_gpu_matches_oracle():
    wl, disps = _graph_scene()
    frames = np.arange(len(wl.frames))
    ii, jj = graph.build_backend_graph(wl.poses0, disps, wl.intr0, frames, beta=0.7, window=10,
                                       max_edges=40, loops=[(0, 13)])
    D = OG.distance_matrix(wl.poses0, disps, wl.intr0, frames, beta=0.7)
    assert list(zip(ii.tolist(), jj.tolist())) == OG.backend_edges(frames, D, 10, 40, [(0, 13)])
