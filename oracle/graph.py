"""Frame-graph construction oracle — TEST INFRASTRUCTURE ONLY.

Restates the map_state operations of ``/root/reference/SPEC.md:134-169`` that produce
the BA edge lists ii/jj.  The reference ships no code for them (``flowsplat`` has only
geometry/providers), so the conventions below are this build's, recorded in DESIGN.md
§Graph (G1-G4) and used identically by ``csrc/dba_graph.cu``:

G1  mean_flow_distance(a, b, beta) (design decision :180):
    beta * mean|flow_full| + (1 - beta) * mean|flow_rot| where, for every pixel p of
    frame a with disparity d (> 0), flow_full = pi(G_ab X) - p with X = unproject(p, d)
    (geometry.py:253-262) and flow_rot = pi(R_ab q) - p with q = ((u-cx)/fx, (v-cy)/fy, 1)
    (translation dropped).  G_ab = G_b o G_a^-1 (providers.py:327).  Evaluated in the
    homogeneous form X~ = R q + t d (Z > Z_MIN <=> Z~ > Z_MIN d) with the flow taken in
    normalised coordinates, du = fx (X~/Z~ - x), so identical frames give exactly 0.
    A pixel counts when its point is in front of the camera (geometry.py:17); image bounds
    are not required (the flow magnitude is defined off-image too).  Each mean is over
    its own valid pixels; no valid pixel -> +inf.
G2  Fixed arithmetic: R = quat_to_matrix (geometry.py:35-41) per pose, R_ab = R_b R_a^T,
    t_ab = t_b - R_ab t_a, every sum left to right, no fused multiply-add; pixel sums run
    over 32 lanes (lane l takes p = l, l+32, ...) then a halving tree (l + 16, 8, 4, 2,
    1).  This makes the GPU kernel and this restatement bitwise equal.
G3  build_frontend_edges(window, radius, ages, max_age):
    every ordered pair of window keyframes at most `radius` apart in window order, plus
    existing edges with both endpoints in the window; an edge with any existing record
    older than max_age (30, Supp. §1.1) is dropped.  Output sorted by (i, j).
G4  build_backend_graph(frames, D, window=150, max_edges=1500, loops):
    the last `window` keyframes; unordered pairs {a<b} ranked by
    (0.5 (D[a,b] + D[b,a]), a, b) ascending (non-finite distances excluded); each pair
    contributes (a,b) and (b,a); loop edges are always kept and count toward the cap; a
    pair is taken only if all of its new edges fit under max_edges, and ranking stops
    at the first pair that does not fit.  Output sorted by (i, j).
"""

from __future__ import annotations

import numpy as np

Z_MIN = 1e-4  # geometry.py:17
LANES = 32


def quat_to_matrix(q):
    """geometry.py:35-41, element by element."""
    w, x, y, z = (float(v) for v in q)
    return np.array([
        [1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
        [2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)],
        [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)],
    ])


def relative(pa, pb):
    """G_ab = G_b o G_a^-1 as (R_ab, t_ab), G2 order (no FMA)."""
    Ra = quat_to_matrix(pa[:4])
    Rb = quat_to_matrix(pb[:4])
    ta = [float(v) for v in pa[4:7]]
    tb = [float(v) for v in pb[4:7]]
    R = np.empty((3, 3))
    for r in range(3):
        for c in range(3):
            R[r, c] = (Rb[r, 0] * Ra[c, 0] + Rb[r, 1] * Ra[c, 1]) + Rb[r, 2] * Ra[c, 2]
    t = np.array([tb[r] - ((R[r, 0] * ta[0] + R[r, 1] * ta[1]) + R[r, 2] * ta[2]) for r in range(3)])
    return R, t


def lane_sum(v):
    """G2 reduction of a per-pixel vector: 32 sequential lane partials, halving tree."""
    n = len(v)
    pad = (-n) % LANES
    rows = np.concatenate([v, np.zeros(pad)]).reshape(-1, LANES)
    acc = np.zeros(LANES)
    for r in rows:
        acc = acc + r
    m = LANES
    while m > 1:
        m //= 2
        acc = acc[:m] + acc[m:2 * m]
    return float(acc[0])


def flow_terms(pose_a, pose_b, disp_a, intr):
    """(sum|flow_full|, n_full, sum|flow_rot|, n_rot) over the pixels of frame a (G1/G2)."""
    H, W = disp_a.shape
    fx, fy, cx, cy = (float(v) for v in intr)
    R, t = relative(pose_a, pose_b)
    p = np.arange(H * W)
    u = (p % W).astype(np.float64)
    v = (p // W).astype(np.float64)
    d = disp_a.reshape(-1).astype(np.float64)
    x = (u - cx) / fx
    y = (v - cy) / fy
    # homogeneous point X~ = R q + t d (q = (x, y, 1)); flows in normalised coordinates
    # scaled by f, so that identical frames give exactly zero
    Xr = (R[0, 0] * x + R[0, 1] * y) + R[0, 2]
    Yr = (R[1, 0] * x + R[1, 1] * y) + R[1, 2]
    Zr = (R[2, 0] * x + R[2, 1] * y) + R[2, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        Xh = Xr + t[0] * d
        Yh = Yr + t[1] * d
        Zh = Zr + t[2] * d
        ok = (d > 0) & (Zh > Z_MIN * d)
        du = fx * (Xh / Zh - x)
        dv = fy * (Yh / Zh - y)
        mf = np.where(ok, np.sqrt(du * du + dv * dv), 0.0)
        okr = Zr > Z_MIN
        dur = fx * (Xr / Zr - x)
        dvr = fy * (Yr / Zr - y)
        mr = np.where(okr, np.sqrt(dur * dur + dvr * dvr), 0.0)
    return lane_sum(mf), int(ok.sum()), lane_sum(mr), int(okr.sum())


def mean_flow_distance(pose_a, pose_b, disp_a, intr, beta=0.5):
    """G1."""
    sf, nf, sr, nr = flow_terms(pose_a, pose_b, disp_a, intr)
    mf = sf / nf if nf > 0 else np.inf
    mr = sr / nr if nr > 0 else np.inf
    return beta * mf + (1.0 - beta) * mr


def distance_matrix(poses, disps, intr, frames, beta=0.5):
    """D[a, b] = mean_flow_distance(frames[a] -> frames[b]); diagonal 0."""
    n = len(frames)
    D = np.zeros((n, n))
    for a in range(n):
        for b in range(n):
            if a != b:
                D[a, b] = mean_flow_distance(poses[frames[a]], poses[frames[b]], disps[frames[a]],
                                             intr, beta)
    return D


def frontend_edges(window, radius=3, existing=(), ages=None, max_age=30):
    """G3."""
    window = [int(k) for k in window]
    inwin = set(window)
    cand = set()
    for a in range(len(window)):
        for b in range(a + 1, min(len(window), a + radius + 1)):
            cand.add((window[a], window[b]))
            cand.add((window[b], window[a]))
    for e in existing:
        e = (int(e[0]), int(e[1]))
        if e[0] in inwin and e[1] in inwin and e[0] != e[1]:
            cand.add(e)
    old = set()
    if ages is not None:
        old = {(int(e[0]), int(e[1])) for e, g in zip(existing, ages) if int(g) > max_age}
    return sorted(e for e in cand if e not in old)


def backend_edges(frames, D, window=150, max_edges=1500, loops=()):
    """G4.  frames: keyframe ids (ascending) indexing D's rows/cols."""
    frames = [int(k) for k in frames]
    n = len(frames)
    w0 = max(0, n - window)
    chosen = set((int(i), int(j)) for i, j in loops)
    keys = []
    for a in range(w0, n):
        for b in range(a + 1, n):
            m = 0.5 * (D[a, b] + D[b, a])
            if np.isfinite(m):
                keys.append((m, frames[a], frames[b]))
    keys.sort()
    for _, i, j in keys:
        new = [e for e in ((i, j), (j, i)) if e not in chosen]
        if len(chosen) + len(new) > max_edges:
            break
        chosen.update(new)
    return sorted(chosen)
