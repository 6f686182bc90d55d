"""Pin the DBA oracle (oracle/dba.py) with the SPEC's own properties.

The reference ships no dba module, so these are the pins (SPEC.md:304-330, 367-371,
807-813): analytic Jacobians vs central finite differences (AC2), Schur solve ==
dense joint solve (AC3, incl. the gauge constraint, intrinsics and the prior),
energy examples (w = 0, zero at truth, alpha = 0), gauge invariance, the zero-step
fixed point at truth, a monotone energy trace and the 8-keyframe recovery (AC1).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import dba as O
from oracle import geometry as G
from tests.helpers import oracle_problem, oracle_state, small_workload


@pytest.fixture(scope="module")
def tiny():
    return small_workload(trajectory="line", frames=3, height=8, width=8, radius=1)


@pytest.fixture(scope="module")
def c1():
    return small_workload("C1")


def _residual(state, prob, e):
    i, j = int(prob.ii[e]), int(prob.jj[e])
    _, h, w = state.disps.shape
    rel = G.relative_pose(state.poses, i, j)
    px, _ = G.reproject(state.disps[i], rel, state.intr)
    return prob.flow[e].reshape(-1, 4)[:, :2].astype(np.float64) - px.reshape(-1, 2)


@pytest.mark.parametrize("calib", [False, True])
def test_jacobians_vs_finite_differences(c1, calib):
    """AC2: analytic J within 1e-4 relative of central differences."""
    st = oracle_state(c1)
    prob = oracle_problem(c1)
    h = 1e-6
    for e in (0, 7, 19):
        r, wt, Ji, Jj, Jd, Jt = O.edge_terms(st, prob, e, calib)
        ok = wt.sum(axis=1) > 0
        i, j = int(prob.ii[e]), int(prob.jj[e])

        def fd(mutate):
            sp, sm = st.copy(), st.copy()
            mutate(sp, +h)
            mutate(sm, -h)
            # projection derivative = -(residual derivative)
            return -(_residual(sp, prob, e) - _residual(sm, prob, e)) / (2 * h)

        for k in range(6):
            xi = np.zeros(6)
            xi[k] = 1.0
            numj = fd(lambda s, eps: s.poses.__setitem__(j, G.retract(s.poses[j], eps * xi)))
            numi = fd(lambda s, eps: s.poses.__setitem__(i, G.retract(s.poses[i], eps * xi)))
            for num, ana in ((numj, Jj[:, :, k]), (numi, Ji[:, :, k])):
                err = np.abs(num[ok] - ana[ok]).max() / max(np.abs(ana[ok]).max(), 1e-12)
                assert err < 1e-4, (e, k, err)
        p = int(np.flatnonzero(ok)[len(np.flatnonzero(ok)) // 2])
        H, W = st.disps.shape[1:]

        def bump(s, eps):
            s.disps[i].reshape(-1)[p] += eps
        numd = fd(bump)[p]
        assert np.allclose(numd, Jd[p], rtol=1e-4, atol=1e-6 * np.abs(Jd[p]).max())
        if calib:
            for k in range(4):
                def bt(s, eps, k=k):
                    s.intr[k] += eps
                numt = fd(bt)
                err = np.abs(numt[ok] - Jt[ok][:, :, k]).max() / max(np.abs(Jt[ok][:, :, k]).max(), 1e-12)
                assert err < 1e-4, (e, k, err)


@pytest.mark.parametrize("calib,gauge,prior", [(False, False, False), (False, None, False),
                                                (True, None, False), (False, False, True)])
def test_schur_equals_dense(tiny, calib, gauge, prior):
    """AC3: Schur complement solve == dense joint solve within 1e-8."""
    wl = tiny
    pr = None
    if prior:
        pr = (wl.true_disps * 1.1).astype(np.float32)
    prob = O.Problem(wl.ii, wl.jj, wl.flow, wl.fixed, pr,
                     None if pr is None else np.ones_like(pr, dtype=np.uint8))
    opts = O.Options(optimize_intrinsics=calib, scale_gauge=gauge)
    st = oracle_state(wl)
    a, da = O.schur_step(st, prob, opts, 1e-4)
    b, db = O.dense_joint_step(st, prob, opts, 1e-4)
    assert np.abs(a - b).max() <= 1e-8 * max(1.0, np.abs(b).max())
    assert np.abs(da - db).max() <= 1e-8 * max(1.0, np.abs(db).max())


def test_energy_examples(c1):
    st = oracle_state(c1)
    prob = oracle_problem(c1)
    zero = prob.flow.copy()
    zero[..., 2:] = 0.0
    assert O.energy(st, O.Problem(prob.ii, prob.jj, zero, prob.fixed)) == 0.0  # w = 0
    truth = O.State(c1.true_poses.copy(), c1.true_disps.copy(), c1.true_intr.copy())
    e0 = O.energy(st, prob)
    assert O.energy(truth, prob) < 1e-10 * e0  # zero at truth (float32 flow rounding only)
    pr = O.Problem(prob.ii, prob.jj, prob.flow, prob.fixed, c1.true_disps.astype(np.float32),
                   np.ones(c1.true_disps.shape, np.uint8))
    assert O.energy(st, pr, O.Options(alpha=0.0)) == pytest.approx(e0, rel=1e-12)  # alpha = 0


def test_gauge_invariance(c1):
    """left-composing every pose with a rigid transform keeps the energy."""
    st = oracle_state(c1)
    prob = oracle_problem(c1)
    T = G.se3_exp(np.array([0.3, -0.2, 0.5, 0.1, 0.2, -0.3]))
    moved = st.copy()
    for k in range(len(moved.poses)):
        # world -> camera poses: a world change X -> T X maps G_k to G_k T^-1
        moved.poses[k] = G.pose_compose(st.poses[k], G.pose_inverse(T))
    assert O.energy(moved, prob) == pytest.approx(O.energy(st, prob), rel=1e-10)


def test_fixed_point_at_truth(c1):
    truth = O.State(c1.true_poses.copy(), c1.true_disps.copy(), c1.true_intr.copy())
    prob = oracle_problem(c1)
    out, rep = O.solve(truth, prob, O.Options(iters=2))
    assert rep.final_energy <= rep.initial_energy + 1e-12
    assert np.abs(out.disps - truth.disps).max() / truth.disps.min() < 1e-6
    assert max(np.linalg.norm(a[4:] - b[4:]) for a, b in zip(out.poses, truth.poses)) < 1e-6


def test_monotone_trace_and_recovery(c1):
    """AC1: 8-keyframe problem recovers the poses within 1e-3
    (relative to the scene diameter, after similarity alignment); energy trace
    non-increasing."""
    st = oracle_state(c1)
    prob = oracle_problem(c1)
    out, rep = O.solve(st, prob, O.Options(iters=6))
    tr = [rep.initial_energy] + rep.energy_trace
    assert all(b <= a for a, b in zip(tr, tr[1:]))
    assert rep.final_energy < 1e-6 * rep.initial_energy
    centers = np.stack([-(G.pose_R(p).T @ p[4:]) for p in out.poses])
    truth = np.stack([-(G.pose_R(p).T @ p[4:]) for p in c1.true_poses])
    # similarity (scale) alignment about camera 0, which is fixed
    a, b = centers - centers[0], truth - truth[0]
    s = float(np.sum(a * b) / np.sum(a * a))
    diam = np.max(np.linalg.norm(truth[:, None] - truth[None], axis=-1))
    assert np.max(np.linalg.norm(s * a - b, axis=1)) < 1e-3 * diam
    for p, q in zip(out.poses, c1.true_poses):
        assert G.rotation_angle_deg(p[:4], q[:4]) < 0.05


def test_fixed_pose_never_moves(c1):
    out, _ = O.solve(oracle_state(c1), oracle_problem(c1), O.Options(iters=2))
    assert np.array_equal(out.poses[0], c1.poses0[0])


def test_nonfinite_raises_with_edge(c1):
    prob = oracle_problem(c1)
    flow = prob.flow.copy()
    flow[5, 3, 4, 0] = np.nan
    flow[5, 3, 4, 2] = 1.0
    with pytest.raises(O.OracleNumericalError) as ei:
        O.solve(oracle_state(c1), O.Problem(prob.ii, prob.jj, flow, prob.fixed), O.Options(iters=1))
    assert ei.value.edge == 5
