"""float64 restatement of flowsplat.geometry — oracle side (test infrastructure).

Conventions (reference ``geometry.py:1-9``): poses are world->camera, stored here
as a flat 7-vector ``[qw, qx, qy, qz, tx, ty, tz]``; se(3) tangents are
``(v, w)`` translation first; pixels are ``(u, v) = (column, row)`` with pixel
centres at integers; depth is parameterised as disparity.

Pinned by tests/test_oracle_geometry.py against the reference's own unit tests
(``pkg/tests/test_geometry.py``) and golden vectors generated from the
reference in ``tests/golden/geometry_golden.npz``.
"""

from __future__ import annotations

import numpy as np

Z_MIN = 1e-4  # geometry.py:17
BOUND_EPS = 1e-9  # geometry.py:247


def hat(w):
    """Skew-symmetric matrix [w]x (geometry.py:68-69)."""
    x, y, z = w
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def qmul(a, b):
    """Hamilton product, (w,x,y,z) storage (geometry.py:24-32)."""
    a0, a1, a2, a3 = a
    b0, b1, b2, b3 = b
    return np.array([
        a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3,
        a0 * b1 + a1 * b0 + a2 * b3 - a3 * b2,
        a0 * b2 - a1 * b3 + a2 * b0 + a3 * b1,
        a0 * b3 + a1 * b2 - a2 * b1 + a3 * b0,
    ])


def qmat(q):
    """Rotation matrix of a unit quaternion (geometry.py:35-41)."""
    w, x, y, z = q
    xx, yy, zz = x * x, y * y, z * z
    return np.array([
        [1 - 2 * (yy + zz), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (xx + zz), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (xx + yy)],
    ])


def mat2q(R):
    """Shepperd's method with sign canonicalised to w >= 0 (geometry.py:44-65)."""
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = 2.0 * np.sqrt(tr + 1.0)
        q = np.array([0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s,
                      (R[1, 0] - R[0, 1]) / s])
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = 2.0 * np.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2])
        q = np.array([(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s,
                      (R[0, 2] + R[2, 0]) / s])
    elif R[1, 1] > R[2, 2]:
        s = 2.0 * np.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2])
        q = np.array([(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s,
                      (R[1, 2] + R[2, 1]) / s])
    else:
        s = 2.0 * np.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1])
        q = np.array([(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s,
                      (R[1, 2] + R[2, 1]) / s, 0.25 * s])
    if q[0] < 0:
        q = -q
    return q / np.linalg.norm(q)


# ---------------------------------------------------------------- poses (7-vectors)

def pose_R(p):
    return qmat(p[:4] / np.linalg.norm(p[:4]))


def pose_compose(a, b):
    """a o b (geometry.py:91-94): quaternion product, renormalised, t = R_a t_b + t_a."""
    q = qmul(a[:4], b[:4])
    q = q / np.linalg.norm(q)
    t = pose_R(a) @ b[4:] + a[4:]
    return np.concatenate([q, t])


def pose_inverse(a):
    """geometry.py:96-99."""
    qi = a[:4] * np.array([1.0, -1.0, -1.0, -1.0])
    qi = qi / np.linalg.norm(qi)
    return np.concatenate([qi, -(qmat(qi) @ a[4:])])


def pose_apply(a, pts):
    return pts @ pose_R(a).T + a[4:]


def relative_pose(poses, i, j):
    """G_ij = G_j o G_i^-1 — the convention fixed by providers.py:327."""
    return pose_compose(poses[j], pose_inverse(poses[i]))


def so3_exp(w):
    """geometry.py:115-122 (small-angle branch below 1e-8)."""
    th = np.linalg.norm(w)
    W = hat(w)
    if th < 1e-8:
        return np.eye(3) + W + 0.5 * (W @ W)
    return np.eye(3) + (np.sin(th) / th) * W + ((1.0 - np.cos(th)) / th**2) * (W @ W)


def so3_left_jacobian(w):
    """geometry.py:125-132 (small-angle branch below 1e-6)."""
    th = np.linalg.norm(w)
    W = hat(w)
    if th < 1e-6:
        return np.eye(3) + 0.5 * W + (W @ W) / 6.0
    return (np.eye(3) + ((1.0 - np.cos(th)) / th**2) * W
            + ((th - np.sin(th)) / th**3) * (W @ W))


def so3_left_jacobian_inv(w):
    """geometry.py:135-142."""
    th = np.linalg.norm(w)
    W = hat(w)
    if th < 1e-6:
        return np.eye(3) - 0.5 * W + (W @ W) / 12.0
    half = 0.5 * th
    return np.eye(3) - 0.5 * W + ((1.0 - half / np.tan(half)) / th**2) * (W @ W)


def se3_exp(xi):
    """(v, w) -> 7-vector pose (geometry.py:145-151)."""
    xi = np.asarray(xi, dtype=np.float64)
    R = so3_exp(xi[3:])
    t = so3_left_jacobian(xi[3:]) @ xi[:3]
    return np.concatenate([mat2q(R), t])


def so3_log(R):
    """geometry.py:154-172."""
    c = np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0)
    th = np.arccos(c)
    vee = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if th < 1e-8:
        return vee / 2.0
    if np.pi - th < 1e-6:
        A = (R + np.eye(3)) / 2.0
        diag = np.sqrt(np.maximum(np.diag(A), 0.0))
        k = int(np.argmax(diag))
        axis = A[:, k] / max(diag[k], 1e-12)
        axis = axis / np.linalg.norm(axis)
        if vee @ axis < 0:
            axis = -axis
        return th * axis
    return th / (2.0 * np.sin(th)) * vee


def se3_log(p):
    """geometry.py:175-178."""
    w = so3_log(pose_R(p))
    return np.concatenate([so3_left_jacobian_inv(w) @ p[4:], w])


def retract(p, xi):
    """Left retraction G <- exp(xi) o G (geometry.py:181-184)."""
    return pose_compose(se3_exp(xi), p)


def rotation_angle_deg(qa, qb):
    """geometry.py:187-192."""
    qa = np.asarray(qa, dtype=np.float64)
    qb = np.asarray(qb, dtype=np.float64)
    qa = qa / np.linalg.norm(qa)
    qb = qb / np.linalg.norm(qb)
    d = np.clip(abs(float(qa @ qb)), 0.0, 1.0)
    return float(np.degrees(2.0 * np.arccos(d)))


def adjoint(p):
    """6x6 adjoint of a pose for (v, w) ordering: exp(Ad xi) = G exp(xi) G^-1."""
    R = pose_R(p)
    A = np.zeros((6, 6))
    A[:3, :3] = R
    A[:3, 3:] = hat(p[4:]) @ R
    A[3:, 3:] = R
    return A


# ---------------------------------------------------------------- pinhole

def pixel_grid(h, w):
    """(H, W, 2) (u, v) grid (geometry.py:228-232)."""
    u, v = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    return np.stack([u, v], axis=-1)


def project(pts, intr, width, height, z_min=Z_MIN):
    """geometry.py:235-250: closed image bounds [0, W] x [0, H] with eps 1e-9."""
    fx, fy, cx, cy = intr
    z = pts[..., 2]
    zs = np.where(np.abs(z) > 1e-300, z, 1e-300)
    u = fx * pts[..., 0] / zs + cx
    v = fy * pts[..., 1] / zs + cy
    ok = ((z > z_min) & (u >= -BOUND_EPS) & (u <= width + BOUND_EPS)
          & (v >= -BOUND_EPS) & (v <= height + BOUND_EPS))
    return np.stack([u, v], axis=-1), ok


def unproject(px, disp, intr):
    """geometry.py:253-262."""
    disp = np.asarray(disp, dtype=np.float64)
    if np.any(disp <= 0):
        raise ValueError("unproject requires strictly positive disparity")
    fx, fy, cx, cy = intr
    z = 1.0 / disp
    return np.stack([(px[..., 0] - cx) / fx * z, (px[..., 1] - cy) / fy * z, z], axis=-1)


def reproject(disp, rel, intr):
    """geometry.py:265-276: unproject -> rigid transform -> project."""
    h, w = disp.shape
    pts = unproject(pixel_grid(h, w), disp, intr)
    return project(pose_apply(rel, pts), intr, w, h)
