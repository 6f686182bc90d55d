"""Per-config timing of DBASolver.solve on the BASELINE configs (C1..C5 at 48x64):
device time per call (CUDA events, inputs resident), trials, accepted iterations; clean
and with 0.5 px correspondence noise (tags *n)."""
import json, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2411_17660_b200 import dba, scenes

out = {}
for name, noise in [(n, z) for z in (0.0, 0.5) for n in ("C1", "C2", "C3", "C4", "C5")]:
    wl = scenes.make_workload(name, height=48, width=64, noise=noise)
    cfg = scenes.CONFIGS[name]
    prior = bool(cfg.get("prior", False))
    calib = bool(cfg.get("calib", False))
    s = dba.DBASolver(wl.ii, wl.jj, len(wl.frames), 48, 64, wl.fixed, optimize_intrinsics=calib, use_prior=prior)
    dev = torch.device('cuda')
    P = torch.as_tensor(wl.poses0, device=dev); D = torch.as_tensor(wl.disps0, dtype=torch.float32, device=dev)
    K = torch.as_tensor(wl.intr0, device=dev); F = torch.as_tensor(wl.flow, dtype=torch.float32, device=dev)
    kw = {}
    if prior:
        kw = dict(prior=torch.as_tensor(wl.prior, dtype=torch.float32, device=dev),
                  prior_mask=torch.as_tensor(wl.prior_mask, device=dev))
    it = cfg["iters"]
    for _ in range(3):
        s.solve(P, D, K, F, iters=it, **kw)
    torch.cuda.synchronize()
    ts, reps = [], []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, _, _, rep = s.solve(P, D, K, F, iters=it, **kw)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); reps.append(rep)
    r = reps[-1]
    tag = name + ("n" if noise > 0 else "")
    out[tag] = dict(noise=noise, keyframes=len(wl.frames), edges=len(wl.ii), iters=it, ms_per_call=float(np.median(ts)),
                     trials=r.trials, accepted=r.iterations_run, calib=calib, prior=prior,
                     ms_per_accepted_iter=float(np.median(ts)) / max(r.iterations_run, 1),
                     initial_energy=r.initial_energy, final_energy=r.final_energy)
    print(tag, json.dumps(out[tag]))
json.dump(out, open('/root/repo/gpurun_out/configs.json', 'w'), indent=1)
