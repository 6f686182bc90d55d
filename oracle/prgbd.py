"""P-RGBD block-coordinate descent and motion-only fill-in —
TEST INFRASTRUCTURE ONLY.

Restates ``/root/reference/SPEC.md:340-348`` (solve_prgbd_bcd) and ``:358-366``
(fill_nonkeyframe_poses); the reference has no code for either.  Conventions
(used identically by ``paper_2411_17660_b200/prgbd.py``):

B1  Eq. 5 term alpha sum m (d* - (s_i d + o_i))^2 enters a solve as the Eq. 4 prior
    with d*' = (d* - o_i)/s_i and per-frame weight s_i^2 (same value, same normal
    equations).
B2  one cycle = stage A: (s, o) frozen, oracle.dba.solve over poses + disparities
    (``iters`` accepted steps); stage B: poses frozen — closed-form (s, o) per frame
    (2x2 least squares over the prior mask, s clamped to >= 1e-4, offset re-solved for
    the clamped scale), then one accepted disparity step (all poses fixed).
    Default 2 cycles.
B3  fill_nonkeyframe_poses: a non-keyframe t between keyframes a <= t <= b starts at
    se3_interpolate(G_a, G_b, (t - a)/(b - a)) (geometry.py:181-184) and, when flow
    records (a -> t), (b -> t) are given, is refined by motion-only Gauss-Newton
    (disparities frozen, keyframes fixed).  t equal to a keyframe id takes that pose.
"""

from __future__ import annotations

import numpy as np

from . import dba as O
from . import geometry as G

S_MIN = 1e-4


def fit_affine(disps, prior, mask, scale, offset, s_min=S_MIN):
    """B2 closed form per frame (float64)."""
    s = np.array(scale, dtype=np.float64)
    o = np.array(offset, dtype=np.float64)
    for f in range(len(s)):
        m = mask[f].reshape(-1).astype(bool)
        if not m.any():
            continue
        d = disps[f].reshape(-1)[m].astype(np.float64)
        ds = prior[f].reshape(-1)[m].astype(np.float64)
        a, b, c = float(d @ d), float(d.sum()), float(m.sum())
        dd, dp = float(d @ ds), float(ds.sum())
        det = a * c - b * b
        sv = (c * dd - b * dp) / det if det > 1e-12 * a * c else s[f]
        if not sv >= s_min:
            sv = s_min
        s[f] = sv
        o[f] = (dp - sv * b) / c
    return s, o


def affine_problem(prob: O.Problem, prior, mask, scale, offset, fixed=None):
    """B1: the Eq. 5 term as an Eq. 4 prior with per-frame weights."""
    eff = ((prior.astype(np.float64) - offset[:, None, None]) / scale[:, None, None])
    return O.Problem(prob.ii, prob.jj, prob.flow, prob.fixed if fixed is None else fixed,
                     prior=eff, prior_mask=mask, prior_weight=scale ** 2)


def combined_energy(state, prob, prior, mask, scale, offset, opts):
    return O.energy(state, affine_problem(prob, prior, mask, scale, offset), opts)


def solve_prgbd_bcd(state: O.State, prob: O.Problem, prior, mask, scale=None, offset=None,
                    opts: O.Options | None = None, cycles=2, stage_b_iters=1):
    """B2.  Returns (state, scale, offset, stage energies [after A, after fit, after B]...)."""
    opts = opts or O.Options()
    N = state.poses.shape[0]
    s = np.ones(N) if scale is None else np.array(scale, dtype=np.float64)
    o = np.zeros(N) if offset is None else np.array(offset, dtype=np.float64)
    cur = state.copy()
    trace = [combined_energy(cur, prob, prior, mask, s, o, opts)]
    all_fixed = np.ones(N, dtype=bool)
    for _ in range(cycles):
        cur, _ = O.solve(cur, affine_problem(prob, prior, mask, s, o), opts)
        trace.append(combined_energy(cur, prob, prior, mask, s, o, opts))
        s, o = fit_affine(cur.disps, prior, mask, s, o)
        trace.append(combined_energy(cur, prob, prior, mask, s, o, opts))
        ob = O.Options(**{**opts.__dict__, "iters": stage_b_iters})
        cur, _ = O.solve(cur, affine_problem(prob, prior, mask, s, o, fixed=all_fixed), ob)
        trace.append(combined_energy(cur, prob, prior, mask, s, o, opts))
    return cur, s, o, trace


def two_stage_uncalibrated(state: O.State, prob: O.Problem, prior, mask, opts: O.Options | None = None,
                           calib_iters=8, cycles=2):
    """stage 1 = solve_ba_calib with the Eq. 4 prior (fixed regulariser)
    from the caller's (heuristic) intrinsics; OracleCalibDegenerate propagates (no stage 2);
    stage 2 = solve_prgbd_bcd with the intrinsics frozen."""
    opts = opts or O.Options()
    p1 = O.Problem(prob.ii, prob.jj, prob.flow, prob.fixed, prior=np.asarray(prior, np.float64),
                   prior_mask=mask)
    o1 = O.Options(**{**opts.__dict__, "iters": calib_iters, "optimize_intrinsics": True})
    st1, _ = O.solve(state, p1, o1)
    o2 = O.Options(**{**opts.__dict__, "optimize_intrinsics": False})
    st2, s, o, trace = solve_prgbd_bcd(st1, prob, prior, mask, opts=o2, cycles=cycles)
    return st2, s, o, trace


def interpolate(pa, pb, tau):
    """se3_interpolate (geometry.py:181-184): exp(tau log(G_b G_a^-1)) G_a."""
    delta = G.se3_log(G.pose_compose(pb, G.pose_inverse(pa)))
    return G.pose_compose(G.se3_exp(tau * delta), pa)


def bracket(kf_ids, t):
    """Nearest keyframes a <= t <= b (clamped at the ends)."""
    kf = sorted(int(k) for k in kf_ids)
    below = [k for k in kf if k <= t]
    above = [k for k in kf if k >= t]
    a = below[-1] if below else kf[0]
    b = above[0] if above else kf[-1]
    return a, b


def fill_nonkeyframe_poses(kf_ids, kf_poses, kf_disps, intr, frames, flows=None,
                           opts: O.Options | None = None):
    """B3.  kf_poses (K,7) / kf_disps (K,H,W) in kf_ids order; flows: {(k, t): (H,W,4)}.
    Returns {t: pose (7,)} for every t in frames."""
    opts = opts or O.Options()
    pos = {int(k): n for n, k in enumerate(kf_ids)}
    out, init = {}, {}
    for t in frames:
        t = int(t)
        if t in pos:
            out[t] = np.array(kf_poses[pos[t]], dtype=np.float64)
            continue
        a, b = bracket(kf_ids, t)
        tau = 0.0 if a == b else (t - a) / (b - a)
        init[t] = interpolate(kf_poses[pos[a]], kf_poses[pos[b]], tau)
    refine = [t for t in init if flows is not None and
              all((k, t) in flows for k in set(bracket(kf_ids, t)))]
    for t in init:
        if t not in refine:
            out[t] = init[t]
    if not refine:
        return out
    K = len(kf_ids)
    H, W = kf_disps.shape[1:]
    poses = np.concatenate([np.asarray(kf_poses, np.float64), np.stack([init[t] for t in refine])])
    disps = np.concatenate([np.asarray(kf_disps, np.float64), np.ones((len(refine), H, W))])
    ii, jj, fl = [], [], []
    for n, t in enumerate(refine):
        for k in sorted(set(bracket(kf_ids, t))):
            ii.append(pos[k])
            jj.append(K + n)
            fl.append(flows[(k, t)])
    fixed = np.zeros(K + len(refine), dtype=bool)
    fixed[:K] = True
    prob = O.Problem(np.array(ii), np.array(jj), np.stack(fl).astype(np.float32), fixed,
                     freeze_disparities=True)
    st, _ = O.solve(O.State(poses, disps, np.asarray(intr, np.float64)), prob, opts)
    for n, t in enumerate(refine):
        out[t] = st.poses[K + n]
    return out
