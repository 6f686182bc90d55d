"""Loop closures in the global graph (the backend graph always
keeps retained loop edges).  A loop edge couples poses far apart in frame order; the plan
then orders the reduced blocks by reverse Cuthill-McKee when that narrows the band
(``dba_plan_create``), and the solve must still match the float64 oracle."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import dba as O
from paper_2411_17660_b200 import _lib, scenes
from tests.helpers import oracle_problem, oracle_state, pose_errors

REL = 1e-4


def _plan_info(ii, jj, n, fixed0=True):
    lib = _lib.load()
    ii = np.ascontiguousarray(ii, np.int32)
    jj = np.ascontiguousarray(jj, np.int32)
    fx = np.zeros(n, np.uint8)
    fx[0] = 1 if fixed0 else 0
    d = _lib.ProblemDesc(n, 8, 8, len(ii), ii.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                         jj.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                         fx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 0, 0, -1, 0, 1)
    h = ctypes.c_void_p()
    code = lib.dba_plan_create(ctypes.byref(d), ctypes.byref(h))
    if code != 0:
        return code, None
    info = _lib.PlanInfo()
    lib.dba_plan_get_info(h, ctypes.byref(info))
    lib.dba_plan_destroy(h)
    return 0, info


def _with_loops(n, r, loops):
    ii, jj = scenes.radius_edges(n, r)
    li = [a for a, b in loops] + [b for a, b in loops]
    lj = [b for a, b in loops] + [a for a, b in loops]
    return np.concatenate([ii, li]).astype(np.int32), np.concatenate([jj, lj]).astype(np.int32)


def test_band_ordering_folds_a_ring_closure():
    ii, jj = scenes.radius_edges(300, 5)
    code, info = _plan_info(ii, jj, 300)
    assert code == 0 and info.band_blocks == 10  # a chain keeps its natural order
    ii, jj = _with_loops(300, 5, [(0, 299)])
    code, info = _plan_info(ii, jj, 300)
    assert code == 0 and info.band_blocks <= 20, info.band_blocks  # natural order: 298
    ii, jj = _with_loops(300, 5, [(1, 299)])
    code, info = _plan_info(ii, jj, 300)
    assert code == 0 and info.band_blocks <= 20


def test_band_limit_is_a_capacity_error():
    # a short cycle in the middle of a long chain cannot be folded below kMaxBand (24)
    ii, jj = _with_loops(300, 5, [(10, 60)])
    code, _ = _plan_info(ii, jj, 300)
    assert code == _lib.DBA_ECAPACITY


def _ring_workload(n=60, r=3, H=24, W=32):
    """An orbit sampled over the full circle, so frame n-1 sees frame 0: the radius graph
    plus the closing edges (0, n-1), (1, n-1), (0, n-2) in both directions."""
    sc = scenes.Scene(scenes.SceneSpec(trajectory="orbit", frames=n, height=H, width=W, seed=0))
    fr = list(range(n))
    ii, jj = _with_loops(n, r, [(0, n - 1), (1, n - 1), (0, n - 2)])
    flow = np.stack([sc.flow_record(int(a), int(b)) for a, b in zip(ii, jj)])
    poses0, disps0 = scenes.perturbed_state(sc, fr)
    fixed = np.zeros(n, bool)
    fixed[0] = True
    return scenes.Workload(name="ring", scene=sc, frames=fr, ii=ii, jj=jj, flow=flow, poses0=poses0,
                           disps0=disps0.astype(np.float32), intr0=sc.intr.copy(), fixed=fixed, iters=4)


@pytest.mark.gpu
def test_ring_closure_solve_parity():
    import torch
    from paper_2411_17660_b200 import dba
    if not torch.cuda.is_available():
        pytest.fail("GPU tests require a CUDA device")
    wl = _ring_workload()
    assert wl.flow[-6:, ..., 2].mean() > 0.3  # the closing edges are covisible
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 24, 32, wl.fixed)
    assert s.info.band_blocks < 20  # folded (natural order: 58)
    S, y, e = s.build_system(wl.poses0, wl.disps0, wl.intr0, wl.flow)
    sysm = O.linearize(oracle_state(wl), oracle_problem(wl), O.Options())
    Sr, yr, _ = O.reduced(sysm, oracle_problem(wl), O.Options())
    assert np.linalg.norm(S - Sr) / np.linalg.norm(Sr) < 1e-10
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) < 1e-10
    for n in (1, 3):
        Po, Do, _, rep = s.solve(wl.poses0, wl.disps0, wl.intr0, wl.flow, iters=n)
        ref, rrep = O.solve(oracle_state(wl), oracle_problem(wl), O.Options(iters=n))
        assert rep.iterations_run == rrep.iterations and rep.trials == rrep.trials
        te, ae = pose_errors(Po.cpu().numpy(), ref.poses)
        assert te < REL and ae < np.degrees(REL), (te, ae)
        rel = np.abs(Do.cpu().numpy() - ref.disps) / ref.disps
        assert rel.max() < REL, rel.max()


@pytest.mark.gpu
def test_backend_graph_with_loops_solves():
    """build_backend_graph over 150 keyframes of a closed orbit (<= 1500 edges, loop edges
    kept) fed straight into the solver: parity with the oracle after 2 iterations."""
    import torch
    from paper_2411_17660_b200 import dba, graph
    if not torch.cuda.is_available():
        pytest.fail("GPU tests require a CUDA device")
    H, W, n = 24, 32, 150
    sc = scenes.Scene(scenes.SceneSpec(trajectory="orbit", frames=n, height=H, width=W, seed=0))
    fr = list(range(n))
    poses0, disps0 = scenes.perturbed_state(sc, fr)
    true_p = np.stack([sc.w2c[k] for k in fr])
    true_d = np.stack([sc.disparity(k) for k in fr]).astype(np.float32)
    ii, jj = graph.build_backend_graph(true_p, true_d, sc.intr, fr, loops=[(0, n - 1)])
    edges = list(zip(ii.tolist(), jj.tolist()))
    assert (0, n - 1) in edges and len(edges) <= 1500
    flow = np.stack([sc.flow_record(int(a), int(b)) for a, b in zip(ii, jj)])
    fixed = np.zeros(n, bool)
    fixed[0] = True
    s = dba.DBASolver(ii, jj, n, H, W, fixed)
    Po, Do, _, rep = s.solve(poses0, disps0.astype(np.float32), sc.intr, flow, iters=2)
    prob = O.Problem(ii, jj, flow, fixed)
    ref, rrep = O.solve(O.State(poses0.copy(), disps0.astype(np.float32).astype(np.float64), sc.intr.copy()),
                        prob, O.Options(iters=2))
    assert rep.iterations_run == rrep.iterations
    te, ae = pose_errors(Po.cpu().numpy(), ref.poses)
    assert te < REL and ae < np.degrees(REL), (te, ae)
    rel = np.abs(Do.cpu().numpy() - ref.disps) / ref.disps
    assert rel.max() < REL, rel.max()
