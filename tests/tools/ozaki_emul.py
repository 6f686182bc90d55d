"""Feasibility: the oracle with its Schur fill-in product computed Ozaki-style (per
128-pixel tile, per-column power-of-two scaling, S signed 7-bit digit slices, products
with s + t <= S + 1 accumulated exactly) -- parity vs the committed fixtures."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
import numpy as np
from oracle import dba as O
from tests import test_dba_golden as T

S_SL = int(sys.argv[1]); TILE = 128
tags = sys.argv[2].split(',')


def ozaki_gram(V):
    P, m = V.shape
    out = np.zeros((m, m))
    for t0 in range(0, P, TILE):
        X = V[t0:t0 + TILE]
        mx = np.abs(X).max(axis=0)
        e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) + 1, 0.0)
        x = X / 2.0 ** e
        mag = np.minimum(np.rint(np.abs(x) * 2.0 ** (7 * S_SL)), 2.0 ** (7 * S_SL) - 1).astype(np.int64)
        sg = np.sign(x).astype(np.int64)
        dig = [((mag >> (7 * (S_SL - s))) & 127) * sg for s in range(1, S_SL + 1)]
        acc = np.zeros((m, m))
        for s in range(S_SL):
            for t in range(S_SL):
                if s + t + 2 <= S_SL + 1:
                    acc += 2.0 ** (-7 * (s + t + 2)) * (dig[s].T @ dig[t]).astype(np.float64)
        out += acc * 2.0 ** (e[:, None] + e[None, :])
    return out


_orig = O.linearize


def linearize(state, prob, opts, frames=None, keep_B=False):
    # the original, then swap the exact fill-in for the sliced one
    N = state.poses.shape[0]
    sysm = _orig(state, prob, opts, frames, keep_B)
    offs, order = O.csr_by_source(prob.ii, N)
    calib = opts.optimize_intrinsics
    if prob.freeze_disparities:
        return sysm
    for i in (range(N) if frames is None else frames):
        edges = [int(x) for x in order[offs[i]:offs[i + 1]]]
        if not edges and not calib:
            continue
        U, C, gd, *_ = O._frame_terms(state, prob, opts, i, edges, calib, False)
        idx = O._local_index(N, i, [int(prob.jj[e]) for e in edges])
        Uc = U / C[:, None]
        sysm.S[np.ix_(idx, idx)] += U.T @ Uc
        sysm.y[idx] += Uc.T @ gd
        V = np.concatenate([U, gd[:, None]], axis=1) / np.sqrt(C)[:, None]
        G = ozaki_gram(V)
        m = U.shape[1]
        sysm.S[np.ix_(idx, idx)] -= G[:m, :m]
        sysm.y[idx] -= G[:m, m]
    return sysm


O.linearize = linearize
for tag in tags:
    g = T._load(tag); wl = T._workload(g)
    calib, prior = bool(g["calib"]), bool(g["prior"])
    refs = T._disps(g, wl)
    prob = O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow, fixed=wl.fixed,
                     prior=wl.prior if prior else None, prior_mask=wl.prior_mask if prior else None)
    st = O.State(wl.poses0.astype(np.float64).copy(), wl.disps0.astype(np.float64).copy(), wl.intr0.astype(np.float64).copy())
    t = time.time()
    n = int(g["iters"])
    snaps = []
    res, rep = O.solve(st, prob, O.Options(iters=n, optimize_intrinsics=calib), snapshot=lambda n_, s, r_: snaps.append(s.copy()))
    worst = 0
    for it, s in enumerate(snaps[:n], 1):
        rel = np.abs(s.disps - refs[it - 1]) / refs[it - 1]
        te = max(np.linalg.norm(s.poses[k, 4:] - g[f"poses_{it}"][k, 4:]) / max(np.linalg.norm(g[f"poses_{it}"][k, 4:]), 1e-12) for k in range(len(s.poses)))
        worst = max(worst, rel.max(), te)
        print(f"  {tag} it {it}: disp max {rel.max():.2e} p999 {np.quantile(rel, 0.999):.2e} pose_t {te:.2e}", flush=True)
    print(f"{tag} S={S_SL}: worst {worst:.2e} trials {rep.trials} vs {int(g[f'trials_{n}'])} ({time.time()-t:.0f}s)", flush=True)
