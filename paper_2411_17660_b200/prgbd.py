"""P-RGBD block-coordinate descent and motion-only pose fill-in.

``solve_prgbd_bcd`` alternates, per cycle (default 2):

* stage A — scales/offsets frozen: the GPU Gauss-Newton (``DBASolver.solve``) over poses
  and disparities with the Eq. 5 term entering as the fused pass's prior term,
  d*' = (d* - o_i)/s_i with per-frame weight s_i^2 (``dba_prior_affine``);
* stage B — poses frozen: closed-form per-frame (s_i, o_i) (``dba_fit_affine``, 2x2 least
  squares in float64 on the device, s_i >= 1e-4), then one accepted disparity step from a
  plan with every pose fixed (the same kernels; the reduced system is empty).

``two_stage_uncalibrated``: stage 1 = ``solve_ba_calib`` with the Eq. 4
prior as a fixed regulariser (alpha = 1e-3) from the heuristic f = (H+W)/2 (geometry.py:
222-225) -- a poorly conditioned intrinsics block raises ``CalibrationDegenerateError`` and
stage 2 is not attempted; stage 2 = ``solve_prgbd_bcd`` with the calibrated intrinsics
frozen (bitwise untouched).

``fill_nonkeyframe_poses``: se(3) geodesic interpolation between the
two nearest keyframes (geometry.py:181-184), refined — when flow records keyframe -> frame
exist — by motion-only Gauss-Newton on the GPU: one plan over all non-keyframes with the
disparity block frozen (no Schur fill-in, disparities untouched) and keyframes fixed.

Conventions B1-B3 are stated in ``oracle/prgbd.py`` (the CPU restatement).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from . import geometry as geo
from .dba import DBASolver, _device, _raise_for, _to_dev

S_MIN = 1e-4


def affine_prior(prior, scale, offset, stream=None):
    """B1: (d* - o)/s (N,H,W) float32 and s^2 (N,) float32 on the device."""
    lib = _lib.load()
    PR = prior.contiguous()
    N = PR.shape[0]
    out = torch.empty_like(PR)
    w = torch.empty(N, dtype=torch.float32, device=PR.device)
    st = stream if stream is not None else torch.cuda.current_stream(PR.device)
    _raise_for(lib.dba_prior_affine(N, PR[0].numel(), ctypes.c_void_p(PR.data_ptr()),
                                    ctypes.c_void_p(scale.data_ptr()), ctypes.c_void_p(offset.data_ptr()),
                                    ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                    ctypes.c_void_p(st.cuda_stream)))
    return out, w


def fit_affine(disps, prior, mask, scale, offset, s_min=S_MIN, stream=None):
    """B2 closed form, in place on the (N,) float64 device tensors scale/offset."""
    lib = _lib.load()
    D, PR, M = disps.contiguous(), prior.contiguous(), mask.contiguous()
    st = stream if stream is not None else torch.cuda.current_stream(D.device)
    _raise_for(lib.dba_fit_affine(D.shape[0], D[0].numel(), ctypes.c_void_p(D.data_ptr()),
                                  ctypes.c_void_p(PR.data_ptr()), ctypes.c_void_p(M.data_ptr()),
                                  ctypes.c_void_p(scale.data_ptr()), ctypes.c_void_p(offset.data_ptr()),
                                  float(s_min), ctypes.c_void_p(st.cuda_stream)))
    return scale, offset


def solve_prgbd_bcd(ii, jj, poses, disps, intr, flow, prior, mask, fixed, scale=None, offset=None, *,
                    cycles=2, iters=4, stage_b_iters=1, freeze_poses=False, freeze_structure=False,
                    device=None, **opts):
    """SPEC.md:340-348.  Returns (poses, disps, scale, offset, trace) where trace holds the
    combined energy at the start and after each stage A / affine fit / stage B."""
    dev = _device(device)
    P = _to_dev(poses, torch.float64, dev).clone()
    D = _to_dev(disps, torch.float32, dev).clone()
    K = _to_dev(intr, torch.float64, dev)
    F = _to_dev(flow, torch.float32, dev)
    PR = _to_dev(prior, torch.float32, dev)
    M = _to_dev(mask, torch.uint8, dev)
    N, H, W = D.shape
    s = (torch.ones(N, dtype=torch.float64, device=dev) if scale is None
         else _to_dev(scale, torch.float64, dev).clone())
    o = (torch.zeros(N, dtype=torch.float64, device=dev) if offset is None
         else _to_dev(offset, torch.float64, dev).clone())
    if freeze_poses and freeze_structure:
        return P, D, s, o, []  # both blocks frozen: a no-op
    solver_a = DBASolver(ii, jj, N, H, W, fixed, use_prior=True, device=dev)
    solver_b = DBASolver(ii, jj, N, H, W, np.ones(N, dtype=bool), use_prior=True, device=dev)

    def energy(pp, dd):
        eff, w = affine_prior(PR, s, o)
        return solver_a.energy(pp, dd, K, F, eff, M, prior_weight=w, **opts)

    trace = [energy(P, D)]
    for _ in range(cycles):
        if not freeze_poses:
            eff, w = affine_prior(PR, s, o)
            P, D, _, _ = solver_a.solve(P, D, K, F, eff, M, prior_weight=w, iters=iters, **opts)
            trace.append(energy(P, D))
        if not freeze_structure:
            fit_affine(D, PR, M, s, o)
            trace.append(energy(P, D))
            eff, w = affine_prior(PR, s, o)
            P, D, _, _ = solver_b.solve(P, D, K, F, eff, M, prior_weight=w, iters=stage_b_iters, **opts)
            trace.append(energy(P, D))
    return P, D, s, o, trace


def heuristic_intrinsics(height, width):
    """f = (H + W)/2, principal point at the image centre (geometry.py:222-225)."""
    f = (height + width) / 2.0
    return np.array([f, f, width / 2.0, height / 2.0])


def two_stage_uncalibrated(ii, jj, poses, disps, flow, prior, mask, fixed, intr0=None, *, calib_iters=8,
                           cycles=2, iters=4, device=None, **opts):
    """SPEC.md:349-357.  Returns (poses, disps, intr, scale, offset, trace); ``trace`` is the
    stage-2 BCD trace.  Raises CalibrationDegenerateError from stage 1 (no stage 2)."""
    dev = _device(device)
    D0 = _to_dev(disps, torch.float32, dev)
    N, H, W = D0.shape
    K0 = heuristic_intrinsics(H, W) if intr0 is None else np.asarray(intr0, np.float64)
    PR = _to_dev(prior, torch.float32, dev)
    M = _to_dev(mask, torch.uint8, dev)
    # stage 1: Eq. 3 + Eq. 4 (fixed prior, no scales/offsets), intrinsics as a global block
    s1 = DBASolver(ii, jj, N, H, W, fixed, optimize_intrinsics=True, use_prior=True, device=dev)
    P1, D1, K1, _ = s1.solve(poses, D0, K0, flow, PR, M, iters=calib_iters, **opts)
    # stage 2: P-RGBD (Eq. 5) with the calibrated camera frozen
    K1 = K1.clone()
    P2, D2, sc, off, trace = solve_prgbd_bcd(ii, jj, P1, D1, K1, flow, PR, M, fixed, cycles=cycles,
                                            iters=iters, device=dev, **opts)
    return P2, D2, K1, sc, off, trace


def _bracket(kf_ids, t):
    kf = sorted(int(k) for k in kf_ids)
    below = [k for k in kf if k <= t]
    above = [k for k in kf if k >= t]
    return (below[-1] if below else kf[0]), (above[0] if above else kf[-1])


def interpolate(pa, pb, tau):
    """se3_interpolate (geometry.py:181-184): exp(tau log(G_b G_a^-1)) G_a (host float64)."""
    delta = geo.log_se3(geo.pose_mul(np.asarray(pb, np.float64), geo.pose_inv(np.asarray(pa, np.float64))))
    return geo.pose_mul(geo.exp_se3(tau * delta), np.asarray(pa, np.float64))


def fill_nonkeyframe_poses(kf_ids, kf_poses, kf_disps, intr, frames, flows=None, *, iters=4, device=None,
                           **opts):
    """SPEC.md:358-366.  kf_poses (K,7) / kf_disps (K,H,W) in kf_ids order; flows maps
    (keyframe, frame) -> (H,W,4) flow record.  Returns {frame: pose (7,) float64}."""
    kf_poses = np.asarray(kf_poses, np.float64)
    pos = {int(k): n for n, k in enumerate(kf_ids)}
    out, init = {}, {}
    for t in frames:
        t = int(t)
        if t in pos:
            out[t] = kf_poses[pos[t]].copy()
            continue
        a, b = _bracket(kf_ids, t)
        init[t] = interpolate(kf_poses[pos[a]], kf_poses[pos[b]], 0.0 if a == b else (t - a) / (b - a))
    refine = [t for t in init if flows is not None and all((k, t) in flows for k in set(_bracket(kf_ids, t)))]
    for t in init:
        if t not in refine:
            out[t] = init[t]
    if not refine:
        return out
    dev = _device(device)
    Kn = len(kf_ids)
    D0 = _to_dev(kf_disps, torch.float32, dev)
    H, W = D0.shape[1:]
    poses = np.concatenate([kf_poses, np.stack([init[t] for t in refine])])
    disps = torch.cat([D0, torch.ones((len(refine), H, W), dtype=torch.float32, device=dev)])
    ii, jj, fl = [], [], []
    for n, t in enumerate(refine):
        for k in sorted(set(_bracket(kf_ids, t))):
            ii.append(pos[k])
            jj.append(Kn + n)
            fl.append(flows[(k, t)])
    fixed = np.zeros(Kn + len(refine), dtype=bool)
    fixed[:Kn] = True
    solver = DBASolver(np.array(ii), np.array(jj), Kn + len(refine), H, W, fixed, freeze_disparities=True,
                       device=dev)
    F = torch.as_tensor(np.stack(fl).astype(np.float32), device=dev)
    P, _, _, _ = solver.solve(poses, disps, intr, F, iters=iters, **opts)
    P = P.cpu().numpy()
    for n, t in enumerate(refine):
        out[t] = P[Kn + n]
    return out
