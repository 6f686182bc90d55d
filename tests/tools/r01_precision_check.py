import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import dba as O
from tests.helpers import oracle_problem, oracle_state, small_workload
from paper_2411_17660_b200 import dba

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

cases = [("C3", dict(height=12, width=16, keyframes=40, radius=2)),
         ("C3", dict(height=12, width=16, keyframes=48, radius=3)),
         ("C1", dict()),
         ("C3", dict(height=48, width=64, keyframes=24, radius=5)),
         ("C5", dict(height=24, width=32, keyframes=16, radius=3))]
for name, kw in cases:
    wl = small_workload(name, **kw)
    calib = name == "C5"
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), wl.flow.shape[1], wl.flow.shape[2], wl.fixed,
                      optimize_intrinsics=calib)
    S, y, e = s.build_system(wl.poses0, wl.disps0, wl.intr0, wl.flow)
    opts = O.Options(optimize_intrinsics=calib)
    prob = oracle_problem(wl)
    t = time.time()
    sysm = O.linearize(oracle_state(wl), prob, opts)
    Sr, yr, _ = O.reduced(sysm, prob, opts)
    delta = s.debug_trial(wl.poses0, wl.disps0, wl.intr0, wl.flow, lam=1e-4)[0]
    dref, _ = O.solve_reduced(Sr, yr, 1e-4)
    w, V = np.linalg.eigh(Sr + 1e-4 * np.eye(len(Sr)))
    dS = S - Sr
    proj = V.T @ dS @ V
    ev = np.abs(np.diag(proj)[:4]) / w[:4]
    print('  asym', rel(S, S.T), 'ref asym', rel(Sr, Sr.T), 'eig', w[:3], 'rel err along weakest', ev)
    print(f"{name} {kw} S {rel(S, Sr):.2e} y {rel(y, yr):.2e} delta {rel(delta, dref):.2e}  (oracle {time.time()-t:.1f}s)", flush=True)
