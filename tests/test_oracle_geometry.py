"""Pin the oracle's geometry restatement (oracle/geometry.py) to the reference.

1. golden vectors generated from /root/reference's flowsplat.geometry
   (tests/golden/make_golden.py) — run everywhere;
2. the reference's own unit tests (pkg/tests/test_geometry.py:21-194) restated
   against the oracle functions;
3. a direct comparison with the reference module when it is importable
   (build container only).
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import scipy.linalg

from oracle import geometry as G

GOLD = os.path.join(os.path.dirname(__file__), "golden", "geometry_golden.npz")
RNG = np.random.default_rng(7)


def _rot_equal(q1, q2, tol=1e-12):
    return np.allclose(G.qmat(q1), G.qmat(q2), atol=tol)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_golden_exp_log(gold):
    for t, e7, l6 in zip(gold["tangents"], gold["exp7"], gold["log6"]):
        p = G.se3_exp(t)
        assert _rot_equal(p[:4], e7[:4]) and np.allclose(p[4:], e7[4:], atol=1e-12)
        assert np.allclose(G.se3_log(e7), l6, atol=1e-10)


def test_golden_compose_inverse_apply(gold):
    e7 = gold["exp7"]
    n = len(e7)
    for k in range(n):
        c = G.pose_compose(e7[k], e7[(k + 1) % n])
        assert _rot_equal(c[:4], gold["compose7"][k][:4])
        assert np.allclose(c[4:], gold["compose7"][k][4:], atol=1e-12)
        iv = G.pose_inverse(e7[k])
        assert _rot_equal(iv[:4], gold["inverse7"][k][:4])
        assert np.allclose(iv[4:], gold["inverse7"][k][4:], atol=1e-12)
        assert np.allclose(G.pose_apply(e7[k], gold["points"][k][None])[0], gold["applied"][k], atol=1e-12)
        assert G.rotation_angle_deg(e7[k][:4], e7[(k + 3) % n][:4]) == pytest.approx(
            gold["angles"][k], abs=1e-9)


def test_golden_pinhole(gold):
    intr = gold["intr"]
    w, h = (int(x) for x in gold["size"])
    px, ok = G.project(gold["cam"], intr, w, h)
    assert np.array_equal(ok, gold["proj_ok"])
    assert np.allclose(px, gold["proj"], atol=1e-12)
    unp = G.unproject(gold["proj"][ok], 1.0 / gold["cam"][ok, 2], intr)
    assert np.allclose(unp, gold["unproj"], atol=1e-12)
    rep, rok = G.reproject(gold["disp"], gold["rel7"], intr)
    assert np.array_equal(rok, gold["reproj_ok"])
    assert np.allclose(rep, gold["reproj"], atol=1e-12)


# ---- the reference's own tests (pkg/tests/test_geometry.py), restated ----

def _random_pose(rot_scale=1.0, trans_scale=1.0):
    return G.se3_exp(np.concatenate([RNG.normal(size=3) * trans_scale, RNG.normal(size=3) * rot_scale]))


def test_exp_zero_is_identity():  # :22-25
    p = G.se3_exp(np.zeros(6))
    assert np.allclose(p[:4], [1, 0, 0, 0]) and np.allclose(p[4:], 0)


def test_exp_pure_yaw_pi():  # :27-31
    p = G.se3_exp(np.array([0, 0, 0, 0, 0, np.pi]))
    assert np.allclose(p[4:], 0, atol=1e-12)
    assert np.allclose(G.pose_R(p) @ np.array([1.0, 0, 0]), [-1, 0, 0], atol=1e-12)


def test_log_exp_roundtrip():  # :33-37
    for _ in range(50):
        v = RNG.normal(size=6)
        v = v / np.linalg.norm(v) * RNG.uniform(0, np.pi / 2)
        assert np.allclose(G.se3_log(G.se3_exp(v)), v, atol=1e-9)


def test_exp_matches_matrix_exponential():  # :39-49 (independent scipy oracle)
    for _ in range(20):
        tau = RNG.normal(size=6) * 0.8
        tw = np.zeros((4, 4))
        tw[:3, :3] = G.hat(tau[3:])
        tw[:3, 3] = tau[:3]
        T = scipy.linalg.expm(tw)
        p = G.se3_exp(tau)
        assert np.allclose(G.pose_R(p), T[:3, :3], atol=1e-10)
        assert np.allclose(p[4:], T[:3, 3], atol=1e-10)


def test_compose_inverse_identity():  # :51-56
    for _ in range(20):
        p = _random_pose()
        e = G.pose_compose(G.pose_inverse(p), p)
        assert np.linalg.norm(e[4:]) < 1e-9
        assert G.rotation_angle_deg(e[:4], [1, 0, 0, 0]) < 1e-6


def test_quaternion_stays_unit():  # :58-62
    p = np.array([1.0, 0, 0, 0, 0, 0, 0])
    for _ in range(200):
        p = G.pose_compose(p, _random_pose(rot_scale=0.3))
        assert abs(np.linalg.norm(p[:4]) - 1.0) < 1e-9


def test_pinhole_analytic():  # :97-135
    intr = np.array([100.0, 100.0, 50.0, 50.0])
    px, ok = G.project(np.array([0.0, 0, 1]), intr, 100, 100)
    assert np.allclose(px, [50, 50]) and ok
    px, ok = G.project(np.array([1.0, 0, 2]), intr, 100, 100)
    assert px[0] == pytest.approx(100.0) and ok
    _, ok = G.project(np.array([0.0, 0, -1]), intr, 100, 100)
    assert not ok
    _, ok = G.project(np.array([5.0, 0, 1]), intr, 100, 100)
    assert not ok
    assert np.allclose(G.unproject(np.array([50.0, 50.0]), 0.5, intr), [0, 0, 2])
    assert np.allclose(G.unproject(np.array([150.0, 50.0]), 1.0, intr), [1, 0, 1])
    with pytest.raises(ValueError):
        G.unproject(np.array([50.0, 50.0]), 0.0, intr)
    for _ in range(200):
        p = RNG.uniform([0, 0], [99, 99])
        d = RNG.uniform(0.05, 5.0)
        back, ok = G.project(G.unproject(p, d, intr), intr, 100, 100)
        assert ok and np.allclose(back, p, atol=1e-9)


def test_reproject_identity_and_homography():  # :139-157
    intr = np.array([100.0, 100.0, 50.0, 50.0])
    disp = RNG.uniform(0.2, 2.0, size=(100, 100))
    corr, ok = G.reproject(disp, np.array([1.0, 0, 0, 0, 0, 0, 0]), intr)
    assert ok.all() and np.allclose(corr, G.pixel_grid(100, 100), atol=1e-12)
    disp = np.full((100, 100), 0.5)
    corr, ok = G.reproject(disp, np.array([1.0, 0, 0, 0, 0, 0, -0.5]), intr)
    expect = (G.pixel_grid(100, 100) - [50, 50]) * (2.0 / 1.5) + [50, 50]
    assert np.allclose(corr[ok], expect[ok], atol=1e-9) and ok.sum() > 1000


def test_reproject_scalar_loop():  # :159-178
    intr = np.array([40.0, 44.0, 16.0, 15.0])
    disp = RNG.uniform(0.3, 1.5, size=(30, 32))
    g = _random_pose(rot_scale=0.05, trans_scale=0.1)
    corr, ok = G.reproject(disp, g, intr)
    R, t = G.pose_R(g), g[4:]
    for v in range(0, 30, 3):
        for u in range(0, 32, 3):
            z = 1.0 / disp[v, u]
            pj = R @ np.array([(u - 16.0) / 40.0 * z, (v - 15.0) / 44.0 * z, z]) + t
            if pj[2] <= 1e-4:
                assert not ok[v, u]
                continue
            uu, vv = 40.0 * pj[0] / pj[2] + 16.0, 44.0 * pj[1] / pj[2] + 15.0
            inb = 0 <= uu <= 32 and 0 <= vv <= 30
            assert ok[v, u] == inb
            if inb:
                assert np.allclose(corr[v, u], [uu, vv], atol=1e-9)


def test_against_reference_module(reference_flowsplat):
    geometry, _ = reference_flowsplat
    for _ in range(30):
        t = RNG.normal(size=6)
        a = geometry.se3_exp(t)
        b = G.se3_exp(t)
        assert _rot_equal(a.quat, b[:4]) and np.allclose(a.trans, b[4:], atol=1e-12)
        assert np.allclose(geometry.se3_log(a), G.se3_log(b), atol=1e-10)
