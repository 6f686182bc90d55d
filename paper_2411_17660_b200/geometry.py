"""Host-side pose helpers for the boundary and the synthetic-scene generator.

Poses cross the boundary as ``(N, 7)`` float64 rows ``[qw, qx, qy, qz, tx, ty, tz]``
(world->camera, unit quaternion, translation) — the field layout of
``flowsplat.geometry.SE3Pose`` (``geometry.py:72-81``).  All BA pose math (relative
poses, adjoints, exp-map retraction) runs on the GPU; the helpers here only serve
the adapters and the fixture generator in ``scenes.py``.
"""

from __future__ import annotations

import numpy as np


def quat_to_rot(q):
    """Rotation matrix of unit quaternion(s) (..., 4) (w, x, y, z) -> (..., 3, 3)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    out = np.empty(q.shape[:-1] + (3, 3))
    out[..., 0, 0] = 1 - 2 * (y * y + z * z)
    out[..., 0, 1] = 2 * (x * y - w * z)
    out[..., 0, 2] = 2 * (x * z + w * y)
    out[..., 1, 0] = 2 * (x * y + w * z)
    out[..., 1, 1] = 1 - 2 * (x * x + z * z)
    out[..., 1, 2] = 2 * (y * z - w * x)
    out[..., 2, 0] = 2 * (x * z - w * y)
    out[..., 2, 1] = 2 * (y * z + w * x)
    out[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return out


def rot_to_quat(R):
    """Largest-pivot (Shepperd) conversion, sign fixed to w >= 0 (geometry.py:44-65)."""
    R = np.asarray(R, dtype=np.float64)
    diag = (R[0, 0], R[1, 1], R[2, 2])
    tr = sum(diag)
    if tr > 0:
        s = 2.0 * np.sqrt(1.0 + tr)
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s,
             (R[1, 0] - R[0, 1]) / s]
    else:
        k = 0 if (R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]) else (1 if R[1, 1] > R[2, 2] else 2)
        a, b = (k + 1) % 3, (k + 2) % 3
        s = 2.0 * np.sqrt(1.0 + R[k, k] - R[a, a] - R[b, b])
        q = [0.0] * 4
        q[0] = (R[b, a] - R[a, b]) / s
        q[1 + k] = 0.25 * s
        q[1 + a] = (R[a, k] + R[k, a]) / s
        q[1 + b] = (R[b, k] + R[k, b]) / s
    q = np.array(q)
    if q[0] < 0:
        q = -q
    return q / np.linalg.norm(q)


def qprod(a, b):
    aw, av = a[0], np.asarray(a[1:])
    bw, bv = b[0], np.asarray(b[1:])
    return np.concatenate([[aw * bw - av @ bv], aw * bv + bw * av + np.cross(av, bv)])


def pose_from_Rt(R, t):
    return np.concatenate([rot_to_quat(R), np.asarray(t, dtype=np.float64)])


def pose_rot(p):
    q = np.asarray(p[:4], dtype=np.float64)
    return quat_to_rot(q / np.linalg.norm(q))


def pose_inv(p):
    qc = np.asarray(p[:4], dtype=np.float64) * np.array([1.0, -1.0, -1.0, -1.0])
    qc = qc / np.linalg.norm(qc)
    return np.concatenate([qc, -(quat_to_rot(qc) @ p[4:])])


def pose_mul(a, b):
    q = qprod(a[:4], b[:4])
    return np.concatenate([q / np.linalg.norm(q), pose_rot(a) @ b[4:] + a[4:]])


def pose_act(p, pts):
    return pts @ pose_rot(p).T + p[4:]


def exp_se3(xi):
    """se(3) exponential of a (v, w) 6-vector as a 7-vector pose (geometry.py:145-151)."""
    xi = np.asarray(xi, dtype=np.float64)
    v, w = xi[:3], xi[3:]
    th = float(np.linalg.norm(w))
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    WW = W @ W
    if th < 1e-8:
        R = np.eye(3) + W + 0.5 * WW
    else:
        R = np.eye(3) + np.sin(th) / th * W + (1 - np.cos(th)) / th**2 * WW
    if th < 1e-6:
        V = np.eye(3) + 0.5 * W + WW / 6.0
    else:
        V = np.eye(3) + (1 - np.cos(th)) / th**2 * W + (th - np.sin(th)) / th**3 * WW
    return pose_from_Rt(R, V @ v)


def log_so3(R):
    """Rotation vector of R (geometry.py:154-171, incl. the near-pi branch)."""
    R = np.asarray(R, dtype=np.float64)
    th = float(np.arccos(np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0)))
    sk = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if th < 1e-8:
        return sk / 2.0
    if np.pi - th < 1e-6:
        A = (R + np.eye(3)) / 2.0
        ax = np.sqrt(np.maximum(np.diag(A), 0.0))
        k = int(np.argmax(ax))
        ax = A[:, k] / max(ax[k], 1e-12)
        ax = ax / np.linalg.norm(ax)
        return th * (ax if sk @ ax >= 0 else -ax)
    return th / (2.0 * np.sin(th)) * sk


def log_se3(p):
    """se(3) logarithm (v, w) of a 7-vector pose (geometry.py:174-177)."""
    w = log_so3(pose_rot(p))
    th = float(np.linalg.norm(w))
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    if th < 1e-6:
        Vinv = np.eye(3) - 0.5 * W + W @ W / 12.0
    else:
        Vinv = (np.eye(3) - 0.5 * W +
                (1.0 / th**2) * (1.0 - th * np.sin(th) / (2.0 * (1.0 - np.cos(th)))) * (W @ W))
    return np.concatenate([Vinv @ np.asarray(p[4:], np.float64), w])


def project_points(pts, fx, fy, cx, cy, width, height, z_min=1e-4):
    """Pinhole projection + validity (closed bounds, eps 1e-9; geometry.py:235-250)."""
    z = pts[..., 2]
    zs = np.where(np.abs(z) > 1e-300, z, 1e-300)
    u = fx * pts[..., 0] / zs + cx
    v = fy * pts[..., 1] / zs + cy
    eps = 1e-9
    ok = (z > z_min) & (u >= -eps) & (u <= width + eps) & (v >= -eps) & (v <= height + eps)
    return np.stack([u, v], axis=-1), ok
