"""Dense bundle adjustment on B200 — the drop-in for the reference's ``dba`` module.

The reference package reserves ``flowsplat.dba`` (``pkg/src/flowsplat/__init__.py:8``)
and specifies it in ``SPEC.md:286-394``; the module file itself is absent.  This
module provides that surface on top of ``libdba_b200.so``:

  energy(problem, state)
  solve_ba(problem, state)
  solve_ba_calib(problem, state)
  energy_rgbd(problem, state, prior, a)

plus a tensor-level API (``DBASolver`` / ``gn_solve``) over device tensors:
poses (N,7) float64 [qw,qx,qy,qz,tx,ty,tz] world->camera, disparities (N,H,W)
float32, intrinsics (4,) float64, edges ii/jj (E,) int32 and the per-edge DSPT flow
record (E,H,W,4) float32 [target_u, target_v, weight_u, weight_v].

Errors map onto ``errors.py`` (the same class names as ``flowsplat.errors``).
There is no CPU path: every call runs the sm_100a kernels and raises if the
library or a CUDA device is unavailable.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import (CalibrationDegenerateError, CapacityError, ConfigError, NumericalError,
                     SolverFailure)

DEFAULTS = dict(lambda0=1e-4, lambda_min=1e-8, lambda_max=1e6, eta=1e-4, alpha=1e-3,
                d_min=1e-6, tangent_max=1.0, calib_cond_max=1e8, damping_candidates=0,
                refine=False)


# ----------------------------------------------------------------------------- SPEC types

@dataclass
class BlockFlags:
    """Variable flags per block."""

    poses: bool = True
    disparities: bool = True
    intrinsics: bool = False
    scales_offsets: bool = False


@dataclass
class BAProblem:
    """SPEC ``BAProblem``: edges + CorrespondenceUpdate data, block flags, fixed set,
    damping, iteration budget.

    ``updates`` holds one object per edge with ``.target`` (H,W,2) and ``.weight``
    (H,W,2) — e.g. ``flowsplat.providers.CorrespondenceUpdate`` — or ``flow`` holds
    the packed (E,H,W,4) record directly.
    """

    edges: list
    updates: list | None = None
    flow: object = None
    fixed: tuple = (0,)
    flags: BlockFlags = field(default_factory=BlockFlags)
    damping: float = 1e-4
    iterations: int = 4
    prior: object = None  # (N,H,W) disparity prior d* (energy_rgbd / RGB-D mode)
    prior_mask: object = None  # (N,H,W) validity of the prior
    alpha: float = 1e-3
    scale_gauge: bool | None = None


@dataclass
class BAState:
    poses: object  # list of SE3Pose-like (.quat, .trans) or (N,7) array
    disparities: object  # (N,H,W)
    intrinsics: object  # PinholeIntrinsics-like (.fx,.fy,.cx,.cy) or (4,) array


@dataclass
class BAReport:
    """SPEC ``BAReport`` + solver diagnostics."""

    initial_energy: float
    final_energy: float
    iterations_run: int
    energy_trace: list
    converged: bool
    trials: int = 0
    lambda_final: float = 0.0
    scale: float = 1.0
    calib_condition: float = 0.0


# ----------------------------------------------------------------------------- helpers

def _raise_for(code: int, rep: _lib.Report | None = None):
    if code == _lib.DBA_OK:
        return
    msg = _lib.status_string(code)
    if code == _lib.DBA_EINVAL:
        raise ConfigError(msg)
    if code == _lib.DBA_ECAPACITY:
        raise CapacityError(msg)
    if code == _lib.DBA_ENONFINITE:
        edge = int(rep.bad_edge) if rep is not None else -1
        raise NumericalError(f"{msg} (edge {edge})", edge=edge)
    if code == _lib.DBA_ESOLVER:
        raise SolverFailure(msg)
    if code == _lib.DBA_ECALIB:
        raise CalibrationDegenerateError(msg)
    raise RuntimeError(f"libdba_b200: {msg} (status {code})")


def _device(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("dba: a CUDA device is required (there is no CPU path)")
    return torch.device(device) if device is not None else torch.device("cuda",
                                                                        torch.cuda.current_device())


def _to_dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        if x.device == device and x.dtype == dtype and x.is_contiguous():
            return x
        return x.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype).to(device, non_blocking=True)


def partition(ii, n_frames, nranks):
    """Source-frame partition used for edge sharding (C-ABI ``dba_partition``)."""
    lib = _lib.load()
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    out = np.zeros(nranks + 1, dtype=np.int32)
    code = lib.dba_partition(int(n_frames), int(len(ii)),
                             ii.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(nranks),
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    _raise_for(code)
    return out


# ----------------------------------------------------------------------------- plan

class DBASolver:
    """A DBA plan for one graph (edges, fixed set, block flags, image size).

    Owns the device workspace.  ``solve`` runs the damped Gauss-Newton loop on the
    GPU; ``energy`` evaluates Eq. 2 (+ Eq. 4); ``build_system`` returns the
    Schur-reduced system (test hook).  With ``nranks > 1`` the plan covers this
    rank's source frames and ``flow`` must hold this rank's edges
    (``local_edges`` order); an NCCL communicator joins the ranks.
    """

    def __init__(self, ii, jj, n_frames, height, width, fixed, *, optimize_intrinsics=False,
                 use_prior=False, scale_gauge=None, rank=0, nranks=1, device=None,
                 nccl_comm=None, freeze_disparities=False):
        self.lib = _lib.load()
        self.device = _device(device)
        self.ii = np.ascontiguousarray(ii, dtype=np.int32)
        self.jj = np.ascontiguousarray(jj, dtype=np.int32)
        fx = np.zeros(n_frames, dtype=np.uint8)
        fixed = np.asarray(fixed)
        if fixed.dtype == bool and fixed.shape == (n_frames,):
            fx[:] = fixed
        else:
            fx[np.asarray(list(fixed), dtype=np.int64)] = 1
        self.fixed = fx
        self.n_frames, self.height, self.width = int(n_frames), int(height), int(width)
        self.optimize_intrinsics = bool(optimize_intrinsics)
        self.use_prior = bool(use_prior)
        self.freeze_disparities = bool(freeze_disparities)
        self.rank, self.nranks = int(rank), int(nranks)
        self.nccl_comm = nccl_comm
        desc = _lib.ProblemDesc(
            self.n_frames, self.height, self.width, len(self.ii),
            self.ii.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            self.jj.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            self.fixed.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            int(self.optimize_intrinsics), int(self.use_prior),
            -1 if scale_gauge is None else int(bool(scale_gauge)), self.rank, self.nranks,
            int(self.freeze_disparities))
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            code = self.lib.dba_plan_create(ctypes.byref(desc), ctypes.byref(handle))
        _raise_for(code)
        self._plan = handle
        info = _lib.PlanInfo()
        _raise_for(self.lib.dba_plan_get_info(self._plan, ctypes.byref(info)))
        self.info = info
        le = np.zeros(max(info.n_local_edges, 1), dtype=np.int32)
        _raise_for(self.lib.dba_plan_local_edges(self._plan,
                                                 le.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        self.local_edges = le[:info.n_local_edges]
        self.workspace = torch.empty(int(info.workspace_bytes) + 256, dtype=torch.uint8,
                                     device=self.device)
        self._ws_ptr = (self.workspace.data_ptr() + 255) & ~255

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                self.lib.dba_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    @property
    def frame_range(self):
        return int(self.info.frame_begin), int(self.info.frame_end)

    def _options(self, iters, **kw):
        o = dict(DEFAULTS)
        o.update({k: v for k, v in kw.items() if v is not None})
        return _lib.Options(int(iters), o["lambda0"], o["lambda_min"], o["lambda_max"], o["eta"],
                            o["alpha"], o["d_min"], o["tangent_max"], o["calib_cond_max"],
                            int(o["damping_candidates"]), 1 if o["refine"] else 0)

    def _inputs(self, poses, disps, intr, flow, prior, prior_mask, prior_weight=None):
        dev = self.device
        P = _to_dev(poses, torch.float64, dev)
        D = _to_dev(disps, torch.float32, dev)
        K = _to_dev(intr, torch.float64, dev)
        F = _to_dev(flow, torch.float32, dev)
        N, H, W = self.n_frames, self.height, self.width
        if P.shape != (N, 7) or D.shape != (N, H, W) or K.shape != (4,):
            raise ConfigError(f"state shapes {tuple(P.shape)}, {tuple(D.shape)}, {tuple(K.shape)} "
                              f"do not match the plan (N={N}, H={H}, W={W})")
        if F.shape != (len(self.local_edges), H, W, 4):
            raise ConfigError(f"flow must be (E_local={len(self.local_edges)}, {H}, {W}, 4), "
                              f"got {tuple(F.shape)}")
        PR = PM = None
        if self.use_prior:
            if prior is None:
                raise ConfigError("plan was created with use_prior=True but no prior given")
            PR = _to_dev(prior, torch.float32, dev)
            PM = (_to_dev(prior_mask, torch.uint8, dev) if prior_mask is not None
                  else (PR > 0).to(torch.uint8))
        self._pw = None
        if prior_weight is not None:
            self._pw = _to_dev(prior_weight, torch.float32, dev).reshape(-1)
            if self._pw.shape != (N,):
                raise ConfigError(f"prior_weight must be (N={N},)")
        return P, D, K, F, PR, PM

    def _buffers(self, P, D, K, F, PR, PM, Po=None, Do=None, Ko=None, stream=None):
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        return _lib.Buffers(
            P.data_ptr(), Po.data_ptr() if Po is not None else None, D.data_ptr(),
            Do.data_ptr() if Do is not None else None, K.data_ptr(),
            Ko.data_ptr() if Ko is not None else None, F.data_ptr(),
            PR.data_ptr() if PR is not None else None, PM.data_ptr() if PM is not None else None,
            self._ws_ptr, int(self.info.workspace_bytes), st.cuda_stream,
            self.nccl_comm if self.nccl_comm is not None else None,
            self._pw.data_ptr() if getattr(self, "_pw", None) is not None else None)

    def solve(self, poses, disps, intr, flow, prior=None, prior_mask=None, *, iters=4,
              out=None, stream=None, prior_weight=None, **opts):
        """Damped Gauss-Newton.  Returns (poses', disps', intr', BAReport)
        as device tensors.  ``out`` may supply preallocated (poses, disps, intr).
        ``prior_weight`` (N,) scales alpha per frame (the Eq. 5 affine prior)."""
        P, D, K, F, PR, PM = self._inputs(poses, disps, intr, flow, prior, prior_mask, prior_weight)
        if out is None:
            Po, Do, Ko = torch.empty_like(P), D.clone(), torch.empty_like(K)
        else:
            Po, Do, Ko = out
        buf = self._buffers(P, D, K, F, PR, PM, Po, Do, Ko, stream)
        rep = _lib.Report()
        o = self._options(iters, **opts)
        with torch.cuda.device(self.device):
            code = self.lib.dba_solve(self._plan, ctypes.byref(o), ctypes.byref(buf),
                                      ctypes.byref(rep))
        _raise_for(code, rep)
        report = BAReport(
            initial_energy=rep.initial_energy, final_energy=rep.final_energy,
            iterations_run=rep.iterations,
            energy_trace=[rep.energy_trace[k] for k in range(rep.trace_len)],
            converged=bool(rep.converged), trials=rep.trials, lambda_final=rep.lambda_final,
            scale=rep.scale, calib_condition=rep.calib_condition)
        return Po, Do, Ko, report

    def energy(self, poses, disps, intr, flow, prior=None, prior_mask=None, prior_weight=None,
               **opts):
        P, D, K, F, PR, PM = self._inputs(poses, disps, intr, flow, prior, prior_mask, prior_weight)
        buf = self._buffers(P, D, K, F, PR, PM)
        e = ctypes.c_double()
        o = self._options(0, **opts)
        with torch.cuda.device(self.device):
            code = self.lib.dba_energy(self._plan, ctypes.byref(o), ctypes.byref(buf),
                                       ctypes.byref(e))
        _raise_for(code)
        return float(e.value)

    def build_system(self, poses, disps, intr, flow, prior=None, prior_mask=None, prior_weight=None,
                     **opts):
        """(S, y, energy) of the Schur-reduced system at the given state (float64 host)."""
        P, D, K, F, PR, PM = self._inputs(poses, disps, intr, flow, prior, prior_mask, prior_weight)
        buf = self._buffers(P, D, K, F, PR, PM)
        n = int(self.info.n_reduced)
        S = np.zeros((max(n, 1), max(n, 1)))
        y = np.zeros(max(n, 1))
        e = ctypes.c_double()
        o = self._options(0, **opts)
        dp = ctypes.POINTER(ctypes.c_double)
        with torch.cuda.device(self.device):
            code = self.lib.dba_build_system(self._plan, ctypes.byref(o), ctypes.byref(buf),
                                             S.ctypes.data_as(dp), y.ctypes.data_as(dp),
                                             ctypes.byref(e))
        _raise_for(code)
        return S[:n, :n], y[:n], float(e.value)


    def set_profiling(self, enable=True):
        """Bracket every pass/solve launch with CUDA events (live kernel timing)."""
        _raise_for(self.lib.dba_plan_set_profiling(self._plan, int(bool(enable))))

    def stats(self, reset=False):
        st = _lib.Stats()
        _raise_for(self.lib.dba_plan_get_stats(self._plan, ctypes.byref(st), int(bool(reset))))
        return {"launches": st.launches, "pass_launches": st.pass_launches,
                "solve_launches": st.solve_launches, "pass_ms": st.pass_ms,
                "solve_ms": st.solve_ms, "pass_runs": st.pass_runs,
                "energy_launches": st.energy_launches, "energy_ms": st.energy_ms}

    def debug_trial(self, poses, disps, intr, flow, prior=None, prior_mask=None, *, lam=1e-4,
                    **opts):
        """Test hook: one solve + trial pass from the input state without acceptance.
        Returns (delta, poses_n, disps_n, intr_n, energy_n) as host arrays."""
        P, D, K, F, PR, PM = self._inputs(poses, disps, intr, flow, prior, prior_mask)
        buf = self._buffers(P, D, K, F, PR, PM)
        n = int(self.info.n_reduced)
        delta = np.zeros(max(n, 1))
        pn = np.zeros((self.n_frames, 7))
        dn = np.zeros((self.n_frames, self.height, self.width), dtype=np.float32)
        kn = np.zeros(4)
        e = ctypes.c_double()
        o = self._options(1, **opts)
        dp = ctypes.POINTER(ctypes.c_double)
        with torch.cuda.device(self.device):
            code = self.lib.dba_debug_trial(self._plan, ctypes.byref(o), ctypes.byref(buf),
                                            float(lam), delta.ctypes.data_as(dp),
                                            pn.ctypes.data_as(dp),
                                            dn.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                            kn.ctypes.data_as(dp), ctypes.byref(e))
        _raise_for(code)
        return delta[:n], pn, dn, kn, float(e.value)


_PLAN_CACHE: dict = {}


def get_solver(ii, jj, n_frames, height, width, fixed, **kw) -> DBASolver:
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    jj = np.ascontiguousarray(jj, dtype=np.int32)
    fx = np.zeros(n_frames, dtype=np.uint8)
    fixed = np.asarray(fixed)
    if fixed.dtype == bool and fixed.shape == (n_frames,):
        fx[:] = fixed
    else:
        fx[np.asarray(list(fixed), dtype=np.int64)] = 1
    key = (ii.tobytes(), jj.tobytes(), fx.tobytes(), n_frames, height, width,
           tuple(sorted((k, str(v)) for k, v in kw.items() if k != "nccl_comm")))
    s = _PLAN_CACHE.get(key)
    if s is None:
        s = DBASolver(ii, jj, n_frames, height, width, fx.astype(bool), **kw)
        if len(_PLAN_CACHE) > 32:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = s
    return s


def gn_solve(poses, disps, intr, ii, jj, flow, fixed, *, iters=4, optimize_intrinsics=False,
             prior=None, prior_mask=None, scale_gauge=None, **opts):
    """Tensor API: one ``solve_ba`` call over device (or host) tensors."""
    N, H, W = (int(s) for s in disps.shape)
    s = get_solver(ii, jj, N, H, W, fixed, optimize_intrinsics=optimize_intrinsics,
                   use_prior=prior is not None, scale_gauge=scale_gauge)
    return s.solve(poses, disps, intr, flow, prior, prior_mask, iters=iters, **opts)


# ----------------------------------------------------------------------------- SPEC adapters

def _pack_state(state: BAState):
    p = state.poses
    if isinstance(p, (list, tuple)):
        poses = np.stack([np.concatenate([np.asarray(g.quat, dtype=np.float64),
                                          np.asarray(g.trans, dtype=np.float64)]) for g in p])
    else:
        poses = np.asarray(p.cpu() if isinstance(p, torch.Tensor) else p, dtype=np.float64)
    k = state.intrinsics
    if hasattr(k, "fx"):
        intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
    else:
        intr = np.asarray(k.cpu() if isinstance(k, torch.Tensor) else k, dtype=np.float64)
    return poses, state.disparities, intr


def _pack_flow(problem: BAProblem, H, W):
    if problem.flow is not None:
        return problem.flow
    if problem.updates is None:
        raise ConfigError("BAProblem needs either updates or flow")
    fl = np.empty((len(problem.updates), H, W, 4), dtype=np.float32)
    for e, u in enumerate(problem.updates):
        fl[e, ..., :2] = u.target
        fl[e, ..., 2:] = u.weight
    return fl


def _unpack_state(state: BAState, poses, disps, intr):
    p = state.poses
    pn = poses.cpu().numpy()
    if isinstance(p, (list, tuple)) and len(p) and hasattr(p[0], "quat"):
        cls = type(p[0])
        new_poses = [cls(pn[k, :4], pn[k, 4:]) for k in range(len(pn))]
    else:
        new_poses = pn
    k = state.intrinsics
    kn = intr.cpu().numpy()
    if hasattr(k, "with_params"):
        new_intr = k.with_params(kn)
    else:
        new_intr = kn
    d = state.disparities
    dn = disps if isinstance(d, torch.Tensor) else disps.cpu().numpy().astype(np.float64)
    return BAState(new_poses, dn, new_intr)


def _blocks(problem: BAProblem, calib: bool):
    """BAProblem block flags -> (fixed frames, optimize_intrinsics, freeze_disparities)
    ("exactly the flagged blocks receive updates").  Per-frame scales and
    offsets exist only in the P-RGBD mode (``prgbd.solve_prgbd_bcd``)."""
    fl = problem.flags if problem.flags is not None else BlockFlags()
    if fl.scales_offsets:
        raise ConfigError("scales_offsets is a P-RGBD block: use prgbd.solve_prgbd_bcd")
    if calib and not fl.intrinsics:
        raise ConfigError("solve_ba_calib needs the intrinsics block flagged (SPEC.md:324)")
    return bool(fl.poses), bool(fl.intrinsics), not bool(fl.disparities)


def _run(problem: BAProblem, state: BAState, calib: bool):
    poses, disps, intr = _pack_state(state)
    N, H, W = (int(s) for s in np.shape(disps))
    edges = np.asarray(problem.edges, dtype=np.int32).reshape(-1, 2)
    if len(edges) == 0:
        raise ConfigError("solve_ba needs at least one edge (SPEC.md:315)")
    flow = _pack_flow(problem, H, W)
    use_prior = problem.prior is not None
    move_poses, calib, freeze_d = _blocks(problem, calib)
    fixed = problem.fixed if move_poses else np.ones(N, dtype=bool)  # poses unflagged: all fixed
    if not move_poses and not calib and freeze_d:  # nothing flagged: the state is returned as is
        e = energy(problem, state)
        return state, BAReport(initial_energy=e, final_energy=e, iterations_run=0, energy_trace=[],
                               converged=True)
    s = get_solver(edges[:, 0], edges[:, 1], N, H, W, fixed,
                   optimize_intrinsics=calib, use_prior=use_prior,
                   scale_gauge=problem.scale_gauge, freeze_disparities=freeze_d)
    Po, Do, Ko, rep = s.solve(poses, disps, intr, flow, problem.prior, problem.prior_mask,
                              iters=problem.iterations, lambda0=problem.damping,
                              alpha=problem.alpha)
    return _unpack_state(state, Po, Do, Ko), rep


def solve_ba(problem: BAProblem, state: BAState):
    """damped GN with Schur elimination; returns (state', BAReport).
    Only the blocks flagged in ``problem.flags`` are updated (poses, disparities and, when
    flagged, the intrinsics)."""
    return _run(problem, state, calib=False)


def solve_ba_calib(problem: BAProblem, state: BAState):
    """as solve_ba with the intrinsics as a global block (the intrinsics
    flag is set for the caller when the problem's flags leave it at the default)."""
    if problem.flags is None or problem.flags == BlockFlags():
        problem = BAProblem(**{**problem.__dict__, "flags": BlockFlags(intrinsics=True)})
    return _run(problem, state, calib=True)


def energy(problem: BAProblem, state: BAState) -> float:
    """Eq. 2 energy (plus Eq. 4 when ``problem.prior`` is set)."""
    poses, disps, intr = _pack_state(state)
    N, H, W = (int(s) for s in np.shape(disps))
    edges = np.asarray(problem.edges, dtype=np.int32).reshape(-1, 2)
    s = get_solver(edges[:, 0], edges[:, 1], N, H, W, problem.fixed,
                   use_prior=problem.prior is not None, scale_gauge=False)
    return s.energy(poses, disps, intr, _pack_flow(problem, H, W), problem.prior,
                    problem.prior_mask, alpha=problem.alpha)


def energy_rgbd(problem: BAProblem, state: BAState, prior, alpha=1e-3, mask=None) -> float:
    """Eq. 2 + alpha * sum m (d* - d)^2.  ``mask`` defaults to the
    prior's validity (d* > 0); a missing prior is a configuration error."""
    if prior is None:
        raise ConfigError("energy_rgbd needs the disparity prior d* (SPEC.md:335)")
    if mask is None:
        mask = (np.asarray(prior.cpu() if isinstance(prior, torch.Tensor) else prior) > 0).astype(np.uint8)
    p = BAProblem(edges=problem.edges, updates=problem.updates, flow=problem.flow,
                  fixed=problem.fixed, flags=problem.flags, prior=prior,
                  prior_mask=mask, alpha=alpha)
    return energy(p, state)
