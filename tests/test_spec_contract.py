"""The SPEC ``dba`` contract beyond per-iteration parity:

* BAProblem block flags -- "exactly the flagged blocks receive updates";
* solve_ba_calib -- fx, fy within 1% from the (H+W)/2 heuristic on a translation-rich
  trajectory, cx, cy within 0.5 px, and the pure-rotation degeneracy error;
* calib + Eq. 4 prior together (stage 1 of two_stage_uncalibrated) against the oracle;
* two_stage_uncalibrated: stage 2 never modifies theta, degenerate input
  raises before stage 2;
* the error contract: SolverFailure at maximum damping, energy_rgbd without a prior.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import dba as O
from oracle import prgbd as OB
from paper_2411_17660_b200.errors import CalibrationDegenerateError, ConfigError, SolverFailure
from tests.helpers import oracle_problem, oracle_state, pose_errors, small_workload

REL = 1e-4
HEUR = np.array([56.0, 56.0, 32.0, 24.0])  # (H+W)/2 at 48x64 (geometry.py:222-225)


def _helix():
    return small_workload(trajectory="helix", frames=60, keyframes=40, radius=3, height=48, width=64,
                          focal=64.0)


def _rotate():
    return small_workload(trajectory="rotate", frames=8, keyframes=8, radius=2, height=24, width=32)


def _problem(wl, **kw):
    from paper_2411_17660_b200 import dba
    edges = list(zip(wl.ii.tolist(), wl.jj.tolist()))
    return dba.BAProblem(edges=edges, flow=wl.flow, fixed=tuple(np.flatnonzero(wl.fixed)), **kw)


def _state(wl, intr=None):
    from paper_2411_17660_b200 import dba
    return dba.BAState(wl.poses0.copy(), wl.disps0.copy(), wl.intr0.copy() if intr is None else intr)


# ----------------------------------------------------------------------------- CPU


def test_oracle_rotation_is_degenerate():
    wl = _rotate()
    with pytest.raises(O.OracleCalibDegenerate):
        O.solve(oracle_state(wl), oracle_problem(wl), O.Options(iters=4, optimize_intrinsics=True))


def test_oracle_ac4_focal_recovery():
    """AC4 pinned on the oracle: from the (H+W)/2 heuristic init (56 vs the true
    64, 12.5 % off) on a translation-rich trajectory, solve_ba_calib recovers fx, fy within 1 %
    (a smaller helix than the GPU test, so the CPU suite stays fast)."""
    wl = small_workload(trajectory="helix", frames=40, keyframes=16, radius=3, height=24, width=32,
                        focal=32.0)
    heur = np.array([28.0, 28.0, 16.0, 12.0])  # (H+W)/2 at 24x32 (geometry.py:222-225)
    st = oracle_state(wl)
    st.intr = heur.copy()
    res, rep = O.solve(st, oracle_problem(wl), O.Options(iters=8, optimize_intrinsics=True))
    assert abs(res.intr[0] - 32.0) / 32.0 < 0.01 and abs(res.intr[1] - 32.0) / 32.0 < 0.01, res.intr
    assert rep.energy_trace[-1] < 1e-3 * rep.energy_trace[0]


def test_oracle_solver_failure_at_max_damping():
    wl = small_workload("C1")
    flow = wl.flow.copy()
    flow[..., 2:] *= -1000.0  # a negative-definite system: no damping up to 1e6 makes it SPD
    with pytest.raises(O.OracleSolverFailure):
        O.solve(oracle_state(wl), O.Problem(wl.ii, wl.jj, flow, wl.fixed), O.Options(iters=2))


def test_adapter_config_errors():
    from paper_2411_17660_b200 import dba
    wl = small_workload("C1")
    st = _state(wl)
    with pytest.raises(ConfigError, match="scales_offsets"):
        dba.solve_ba(_problem(wl, flags=dba.BlockFlags(scales_offsets=True)), st)
    with pytest.raises(ConfigError, match="intrinsics"):
        dba.solve_ba_calib(_problem(wl, flags=dba.BlockFlags(poses=True, disparities=False)), st)
    with pytest.raises(ConfigError, match="prior"):
        dba.energy_rgbd(_problem(wl), st, None)


# ----------------------------------------------------------------------------- GPU


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests require a CUDA device")
    return torch


@pytest.mark.gpu
def test_flag_disparities_frozen(cuda):
    from paper_2411_17660_b200 import dba
    wl = small_workload("C1")
    out, rep = dba.solve_ba(_problem(wl, iterations=3, flags=dba.BlockFlags(disparities=False)), _state(wl))
    d = np.asarray(out.disparities)
    assert np.array_equal(d.astype(np.float32), wl.disps0)  # bitwise untouched
    prob = O.Problem(wl.ii, wl.jj, wl.flow, wl.fixed, freeze_disparities=True)
    ref, rrep = O.solve(oracle_state(wl), prob, O.Options(iters=3))
    te, ae = pose_errors(np.asarray(out.poses), ref.poses)
    assert te < REL and ae < np.degrees(REL), (te, ae)
    assert rep.iterations_run == rrep.iterations


@pytest.mark.gpu
def test_flag_poses_frozen(cuda):
    from paper_2411_17660_b200 import dba
    wl = small_workload("C1")
    out, rep = dba.solve_ba(_problem(wl, iterations=2, flags=dba.BlockFlags(poses=False)), _state(wl))
    assert np.array_equal(np.asarray(out.poses), wl.poses0)  # bitwise untouched
    allfix = np.ones(len(wl.frames), dtype=bool)
    ref, rrep = O.solve(oracle_state(wl), O.Problem(wl.ii, wl.jj, wl.flow, allfix), O.Options(iters=2))
    rel = np.abs(np.asarray(out.disparities) - ref.disps) / ref.disps
    assert rel.max() < REL, rel.max()
    assert rep.iterations_run == rrep.iterations


@pytest.mark.gpu
def test_flag_intrinsics_in_solve_ba_matches_calib(cuda):
    from paper_2411_17660_b200 import dba
    wl = small_workload("C5", keyframes=6, radius=2)
    a, ra = dba.solve_ba(_problem(wl, iterations=2, flags=dba.BlockFlags(intrinsics=True)), _state(wl))
    b, rb = dba.solve_ba_calib(_problem(wl, iterations=2), _state(wl))
    assert not np.array_equal(np.asarray(a.intrinsics), wl.intr0)
    assert np.array_equal(np.asarray(a.intrinsics), np.asarray(b.intrinsics))
    assert np.array_equal(np.asarray(a.poses), np.asarray(b.poses))
    # nothing flagged: a no-op
    c, rc = dba.solve_ba(_problem(wl, flags=dba.BlockFlags(poses=False, disparities=False)), _state(wl))
    assert rc.iterations_run == 0 and np.array_equal(np.asarray(c.poses), wl.poses0)


@pytest.mark.gpu
def test_calibration_recovers_focal_lengths(cuda):
    """fx, fy within 1% from the (H+W)/2 heuristic (here 56 vs 64, 12.5% off)
    on a translation-rich trajectory; cx, cy (initialised at the truth) within 0.5 px."""
    from paper_2411_17660_b200 import dba
    wl = _helix()
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 48, 64, wl.fixed, optimize_intrinsics=True)
    _, _, K, rep = s.solve(wl.poses0, wl.disps0, HEUR, wl.flow, iters=8)
    K = K.cpu().numpy()
    assert abs(K[0] - 64.0) / 64.0 < 0.01 and abs(K[1] - 64.0) / 64.0 < 0.01, K
    assert abs(K[2] - 32.0) < 0.5 and abs(K[3] - 24.0) < 0.5, K
    assert rep.final_energy < 1e-6 * rep.initial_energy


@pytest.mark.gpu
def test_calibration_pure_rotation_raises(cuda):
    from paper_2411_17660_b200 import dba
    wl = _rotate()
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 24, 32, wl.fixed, optimize_intrinsics=True)
    with pytest.raises(CalibrationDegenerateError):
        s.solve(wl.poses0, wl.disps0, wl.intr0, wl.flow, iters=4)


@pytest.mark.gpu
def test_solver_failure_at_max_damping(cuda):
    from paper_2411_17660_b200 import dba
    wl = small_workload("C1")
    flow = wl.flow.copy()
    flow[..., 2:] *= -1000.0
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), wl.flow.shape[1], wl.flow.shape[2], wl.fixed)
    with pytest.raises(SolverFailure):
        s.solve(wl.poses0, wl.disps0, wl.intr0, flow, iters=2)


def _calib_prior_wl():
    wl = small_workload("C5", keyframes=8, radius=2)
    prior = np.stack([wl.scene.depth_prior(k) for k in wl.frames]).astype(np.float32)
    return wl, prior, (prior > 0).astype(np.uint8)


@pytest.mark.gpu
def test_calib_with_prior_parity(cuda):
    """Stage 1 of two_stage_uncalibrated: intrinsics + Eq. 4 prior in one reduced system."""
    from paper_2411_17660_b200 import dba
    wl, prior, mask = _calib_prior_wl()
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 24, 32, wl.fixed, optimize_intrinsics=True, use_prior=True)
    S, y, e = s.build_system(wl.poses0, wl.disps0, wl.intr0, wl.flow, prior, mask)
    opts = O.Options(optimize_intrinsics=True)
    prob = O.Problem(wl.ii, wl.jj, wl.flow, wl.fixed, prior=prior, prior_mask=mask)
    sysm = O.linearize(oracle_state(wl), prob, opts)
    Sr, yr, _ = O.reduced(sysm, prob, opts)
    assert np.linalg.norm(S - Sr) / np.linalg.norm(Sr) < 1e-10
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-10
    Po, Do, Ko, rep = s.solve(wl.poses0, wl.disps0, wl.intr0, wl.flow, prior, mask, iters=3)
    ref, rrep = O.solve(oracle_state(wl), prob, O.Options(iters=3, optimize_intrinsics=True))
    assert rep.iterations_run == rrep.iterations and rep.trials == rrep.trials
    te, ae = pose_errors(Po.cpu().numpy(), ref.poses)
    assert te < REL and ae < np.degrees(REL)
    rel = np.abs(Do.cpu().numpy() - ref.disps) / ref.disps
    assert rel.max() < REL, rel.max()
    assert np.max(np.abs(Ko.cpu().numpy() - ref.intr) / ref.intr) < REL


@pytest.mark.gpu
def test_two_stage_uncalibrated(cuda):
    from paper_2411_17660_b200 import prgbd
    wl, prior, mask = _calib_prior_wl()
    K0 = prgbd.heuristic_intrinsics(24, 32)
    P, D, K, sc, off, trace = prgbd.two_stage_uncalibrated(wl.ii, wl.jj, wl.poses0, wl.disps0, wl.flow, prior,
                                                           mask, wl.fixed, K0, calib_iters=4, cycles=1)
    st, rs, ro, rtrace = OB.two_stage_uncalibrated(
        O.State(wl.poses0.copy(), wl.disps0.astype(np.float64), K0.copy()),
        O.Problem(wl.ii, wl.jj, wl.flow, wl.fixed), prior, mask, calib_iters=4, cycles=1)
    assert np.max(np.abs(K.cpu().numpy() - st.intr) / st.intr) < REL
    te, ae = pose_errors(P.cpu().numpy(), st.poses)
    assert te < REL and ae < np.degrees(REL)
    rel = np.abs(D.cpu().numpy() - st.disps) / st.disps
    assert rel.max() < REL, rel.max()
    assert np.allclose(sc.cpu().numpy(), rs, rtol=REL) and np.allclose(off.cpu().numpy(), ro, atol=REL)
    # rotation-only input: the stage-1 degeneracy error, stage 2 never runs
    wr = _rotate()
    pr = np.stack([wr.scene.depth_prior(k) for k in wr.frames]).astype(np.float32)
    with pytest.raises(CalibrationDegenerateError):
        prgbd.two_stage_uncalibrated(wr.ii, wr.jj, wr.poses0, wr.disps0, wr.flow, pr, (pr > 0).astype(np.uint8),
                                     wr.fixed, prgbd.heuristic_intrinsics(24, 32), calib_iters=4)
