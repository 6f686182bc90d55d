"""Shared test helpers: small deterministic DBA problems and oracle adapters."""

from __future__ import annotations

import numpy as np

from oracle import dba as O
from oracle import geometry as OG
from paper_2411_17660_b200 import scenes


def small_workload(name="C1", height=24, width=32, keyframes=None, radius=None, iters=None,
                   trajectory=None, frames=None, focal=None, noise=0.0, seed=0):
    """A reduced-resolution version of a BASELINE config (same scene family)."""
    if trajectory is None:
        return scenes.make_workload(name, height=height, width=width, keyframes=keyframes,
                                    radius=radius, iters=iters)
    spec = scenes.SceneSpec(trajectory=trajectory, frames=frames, height=height, width=width,
                            seed=seed, focal=focal, pixel_noise=noise)
    sc = scenes.Scene(spec)
    fr = list(range(keyframes or frames))
    ii, jj = scenes.radius_edges(len(fr), radius)
    flow = np.stack([sc.flow_record(fr[a], fr[b]) for a, b in zip(ii, jj)])
    poses0, disps0 = scenes.perturbed_state(sc, fr)
    fixed = np.zeros(len(fr), dtype=bool)
    fixed[0] = True
    return scenes.Workload(name=f"{trajectory}{frames}", scene=sc, frames=fr, ii=ii, jj=jj,
                           flow=flow, poses0=poses0, disps0=disps0.astype(np.float32),
                           intr0=sc.intr.copy(), fixed=fixed, iters=iters or 4,
                           true_poses=np.stack([sc.w2c[k] for k in fr]),
                           true_disps=np.stack([sc.disparity(k) for k in fr]),
                           true_intr=sc.intr.copy())


def oracle_problem(wl, fixed=None, prior=False):
    return O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow,
                     fixed=wl.fixed if fixed is None else fixed,
                     prior=wl.prior if prior else None,
                     prior_mask=wl.prior_mask if prior else None)


def oracle_state(wl, poses=None, disps=None, intr=None):
    return O.State(
        (wl.poses0 if poses is None else poses).astype(np.float64).copy(),
        (wl.disps0 if disps is None else disps).astype(np.float64).copy(),
        (wl.intr0 if intr is None else intr).astype(np.float64).copy())


def pose_errors(pa, pb):
    """(max relative translation error, max rotation angle deg) between pose sets."""
    rel = []
    ang = []
    for a, b in zip(pa, pb):
        n = max(np.linalg.norm(b[4:]), 1e-12)
        rel.append(np.linalg.norm(a[4:] - b[4:]) / n)
        ang.append(OG.rotation_angle_deg(a[:4], b[:4]))
    return float(max(rel)), float(max(ang))
