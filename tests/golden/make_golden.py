"""Generate the committed golden fixtures from the REFERENCE implementation.

Run in the build container (needs /root/reference; never run on the GPU box):

    python tests/golden/make_golden.py

Outputs (small, committed):
  geometry_golden.npz  reference flowsplat.geometry outputs on seeded random inputs:
                       se3_exp / se3_log / compose / inverse / apply / project /
                       unproject / reproject / rotation_angle_between
  scene_line6.npz      reference flowsplat.providers.SyntheticProviders output for a
                       small line scene (6 frames, 24x32, radius-2 graph, with pixel
                       noise): poses, disparities, flow records, depth priors
The oracle (oracle/geometry.py) and the scene port (paper_2411_17660_b200/scenes.py)
are pinned against these files by tests/test_oracle_geometry.py and tests/test_scenes.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from flowsplat import geometry as g
    from flowsplat import providers as pr

    rng = np.random.default_rng(20241127)
    n = 64
    tang = rng.normal(size=(n, 6)) * np.array([1.0, 1.0, 1.0, 0.7, 0.7, 0.7])
    exp7 = np.stack([np.concatenate([g.se3_exp(t).quat, g.se3_exp(t).trans]) for t in tang])
    poses = [g.se3_exp(t) for t in tang]
    log6 = np.stack([g.se3_log(p) for p in poses])
    comp = np.stack([np.concatenate([poses[k].compose(poses[(k + 1) % n]).quat,
                                     poses[k].compose(poses[(k + 1) % n]).trans]) for k in range(n)])
    inv = np.stack([np.concatenate([p.inverse().quat, p.inverse().trans]) for p in poses])
    pts = rng.normal(size=(n, 3)) * 2.0
    applied = np.stack([poses[k].apply(pts[k][None])[0] for k in range(n)])
    ang = np.array([g.rotation_angle_between(poses[k], poses[(k + 3) % n]) for k in range(n)])
    intr = g.PinholeIntrinsics(40.0, 44.0, 16.0, 15.0, 32, 30)
    cam = rng.normal(size=(n, 3)) * np.array([1.0, 1.0, 0.5]) + np.array([0, 0, 2.0])
    px, ok = g.project(cam, intr)
    disp = rng.uniform(0.3, 1.5, size=(30, 32))
    rel = g.se3_exp(np.array([0.05, -0.03, 0.1, 0.02, -0.04, 0.03]))
    rep, rep_ok = g.reproject(disp, rel, intr)
    unp = g.unproject(px[ok], 1.0 / cam[ok, 2], intr)
    np.savez_compressed(
        os.path.join(HERE, "geometry_golden.npz"),
        tangents=tang, exp7=exp7, log6=log6, compose7=comp, inverse7=inv, points=pts,
        applied=applied, angles=ang, intr=np.array([40.0, 44.0, 16.0, 15.0]), size=np.array([32, 30]),
        cam=cam, proj=px, proj_ok=ok, disp=disp, rel7=np.concatenate([rel.quat, rel.trans]),
        reproj=rep, reproj_ok=rep_ok, unproj=unp)

    spec = pr.SceneSpec(trajectory="line", frames=6, height=24, width=32, seed=3,
                        pixel_noise=0.05, prior_scale_range=(0.8, 1.2),
                        prior_offset_range=(-0.02, 0.02), prior_noise=0.01)
    sc = pr.SyntheticScene(spec)
    prov = pr.SyntheticProviders(sc)
    ii, jj = [], []
    for i in range(6):
        for j in range(max(0, i - 2), min(6, i + 3)):
            if j != i:
                ii.append(i)
                jj.append(j)
    flow = []
    for i, j in zip(ii, jj):
        u = prov.provide_correspondences(i, j)
        flow.append(np.concatenate([u.target, u.weight], axis=-1).astype(np.float32))
    np.savez_compressed(
        os.path.join(HERE, "scene_line6.npz"),
        ii=np.array(ii, dtype=np.int32), jj=np.array(jj, dtype=np.int32), flow=np.stack(flow),
        w2c=np.stack([np.concatenate([sc.pose_w2c(k).quat, sc.pose_w2c(k).trans]) for k in range(6)]),
        disparity=np.stack([sc.disparity(k) for k in range(6)]),
        prior=np.stack([prov.provide_depth_prior(k) for k in range(6)]),
        intr=sc.intrinsics.as_vector())
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
