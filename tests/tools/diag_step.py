import sys, os, json, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
import numpy as np
from oracle import dba as O
from paper_2411_17660_b200 import scenes, dba
import dba_codec
tag, cfg, noise, it = sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4])
lam = float(sys.argv[5])
wl = scenes.make_workload(cfg, noise=noise)
g = np.load(f'/root/repo/tests/golden/dba_{tag}.npz')
refs = dba_codec.decode(wl.disps0, [g[f'dq_{k}'] for k in range(1, it + 1)])
P1 = g[f'poses_{it}']; D1 = refs[it - 1].astype(np.float32); K1 = g[f'intr_{it}']
calib = bool(g['calib'])
s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 48, 64, wl.fixed, optimize_intrinsics=calib)
S, y, e = s.build_system(P1, D1, K1, wl.flow)
prob = O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow, fixed=wl.fixed)
opts = O.Options(optimize_intrinsics=calib)
st = O.State(P1.copy(), D1.astype(np.float64), K1.copy())
t0 = time.time()
sysm = O.linearize(st, prob, opts)
Sr, yr, _ = O.reduced(sysm, prob, opts)
print('oracle lin', time.time() - t0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print('S rel', rel(S, Sr), 'y rel', rel(y, yr), 'E', e, sysm.energy, (e - sysm.energy) / sysm.energy)
dS = np.abs(S - Sr); print('S max abs diff', dS.max(), 'max |S|', np.abs(Sr).max())
ev = np.linalg.eigvalsh(Sr + lam * np.eye(len(Sr)))
print('eig min/max', ev.min(), ev.max(), 'cond', ev.max() / ev.min())
dref, _ = O.solve_reduced(Sr, yr, lam)
dalt = np.linalg.solve(S + lam * np.eye(len(S)), y)  # oracle solver on the GPU's system
delta, pn, dn, kn, en = s.debug_trial(P1, D1, K1, wl.flow, lam=lam)
print('delta gpu vs oracle', rel(delta, dref), ' oracle-solve(GPU S,y) vs oracle', rel(dalt, dref),
      ' gpu vs oracle-solve(GPU S,y)', rel(delta, dalt))
