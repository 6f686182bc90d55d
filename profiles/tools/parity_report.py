"""Per-iteration GPU-vs-oracle parity on every committed golden fixture (clean and noisy
BASELINE configs at 48x64): max / p99.9 relative disparity error (denominator d_ref),
pose translation / rotation, intrinsics, trial counts, and the worst pixel's context.
Writes gpurun_out/parity.json.   python profiles/tools/parity_report.py [TAG ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from tests import test_dba_golden as T  # noqa: E402
from paper_2411_17660_b200 import dba  # noqa: E402

tags = sys.argv[1:] or T.TAGS
out = {}
for tag in tags:
    g = T._load(tag)
    wl = T._workload(g)
    calib, prior = bool(g["calib"]), bool(g["prior"])
    refs = T._disps(g, wl)
    H, W = int(g["height"]), int(g["width"])
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), H, W, wl.fixed, optimize_intrinsics=calib,
                      use_prior=prior)
    kw = dict(prior=wl.prior, prior_mask=wl.prior_mask) if prior else {}
    rows = []
    for n in range(1, int(g["iters"]) + 1):
        Po, Do, Ko, rep = s.solve(wl.poses0, wl.disps0, wl.intr0, wl.flow, iters=n, **kw)
        D = Do.cpu().numpy().astype(np.float64)
        st = T.parity_stats(Po.cpu().numpy(), D, Ko.cpu().numpy() if calib else None, g, n,
                            refs[n - 1])
        rel = np.abs(D - refs[n - 1]) / refs[n - 1]
        k = int(np.argmax(rel))
        f, p = np.unravel_index(k, rel.shape[:1] + (H * W,))
        dprev = (wl.disps0.astype(np.float64) if n == 1 else refs[n - 2]).reshape(-1)[k]
        st.update(trials=rep.trials, trials_ref=int(g[f"trials_{n}"]), iters_run=rep.iterations_run,
                  n_bad=int(np.count_nonzero(rel >= 1e-4)),
                  energy=rep.final_energy, energy_ref=float(g[f"energy_{n}"][-1]),
                  worst=dict(frame=int(f), pixel=int(p), d=float(D.reshape(-1)[k]),
                             d_ref=float(refs[n - 1].reshape(-1)[k]), d_prev=float(dprev),
                             d_true=float(wl.true_disps.reshape(-1)[k])))
        rows.append(st)
        print(tag, json.dumps(st), flush=True)
    out[tag] = rows
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity.json"), "w"), indent=1)
