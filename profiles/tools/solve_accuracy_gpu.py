# GPU step accuracy: the band solve (dba_debug_trial) against a 3x refined dense Cholesky of
# the same GPU-assembled reduced system (dba_build_system), noisy C3 at golden iterations 0/2/4/8.
# DBA_B200_LIB=<another build> compares a different solver build.
import os, sys, numpy as np, scipy.linalg as sl
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
import torch
from paper_2411_17660_b200 import scenes, dba
import dba_codec
g = np.load('/root/repo/tests/golden/dba_C3n.npz')
wl = scenes.make_workload("C3", height=48, width=64, noise=0.5)
for n in (0, 2, 4, 8):
    if n == 0:
        P, D = wl.poses0, wl.disps0
    else:
        D = dba_codec.decode(wl.disps0, [g[f"dq_{k}"] for k in range(1, n + 1)])[n - 1].astype(np.float32); P = g[f"poses_{n}"]
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 48, 64, wl.fixed)
    S, y, _ = s.build_system(P, D, wl.intr0, wl.flow)
    lam = 1e-4
    A = S + lam * np.eye(S.shape[0]); c = sl.cho_factor(A); x = sl.cho_solve(c, y)
    x0 = x.copy()
    for _ in range(3): x = x + sl.cho_solve(c, y - A @ x)
    delta = s.debug_trial(P, D, wl.intr0, wl.flow, lam=lam)[0]
    print(os.environ.get('DBA_B200_LIB', 'current'), n, 'cond %.1e' % np.linalg.cond(A), 'gpu err %.2e' % (np.abs(delta - x).max() / np.abs(x).max()), 'lapack %.2e' % (np.abs(x0 - x).max() / np.abs(x).max()), flush=True)
