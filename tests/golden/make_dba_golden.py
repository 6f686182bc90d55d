"""Generate committed DBA golden fixtures from the float64 CPU oracle ("committed
.npz golden outputs from the oracle, per config and per iteration, then pin GPU parity").

    python tests/golden/make_dba_golden.py

For each BASELINE config (C1 mono, C2 frontend window, C3 global backend, C4 depth prior,
C5 self-calibrating), at its own 48x64 resolution, the deterministic workload of
``paper_2411_17660_b200.scenes.make_workload`` is solved by ``oracle.dba.solve`` for
1..iters accepted GN iterations, and the state after each is stored (poses and
intrinsics float64, disparities float32 -- 6e-8 relative, far below the 1e-4 bar), with
the energy trace, trial count and a checksum of the inputs.  ``tests/test_dba_golden.py``
re-derives C1 iteration 1 with the oracle (pins the oracle against itself) and compares
the GPU path against every fixture.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import dba as O  # noqa: E402
from paper_2411_17660_b200 import scenes  # noqa: E402

# name -> (config, height, width, keyframes, iterations)
FIXTURES = {
    "C1": ("C1", 48, 64, None, 4),
    "C2": ("C2", 48, 64, None, 2),
    "C3": ("C3", 48, 64, None, 1),  # the bench config itself (first GN iteration)
    "C4": ("C4", 48, 64, None, 2),
    "C5": ("C5", 48, 64, None, 2),
}


def input_checksum(wl):
    h = np.float64(0.0)
    for a in (wl.poses0, wl.disps0, wl.flow, wl.intr0):
        x = np.asarray(a, np.float64).ravel()
        h += np.sum(x * (1.0 + np.arange(x.size) % 7))
    return float(h)


def main():
    for tag, (cfg, H, W, kf, iters) in FIXTURES.items():
        t0 = time.time()
        wl = scenes.make_workload(cfg, height=H, width=W, keyframes=kf)
        calib = bool(wl.optimize_intrinsics)
        prior = wl.prior is not None
        prob = O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow, fixed=wl.fixed,
                         prior=wl.prior if prior else None, prior_mask=wl.prior_mask if prior else None)
        out = dict(config=cfg, height=H, width=W, keyframes=len(wl.frames), iters=iters, calib=calib,
                   prior=prior, checksum=input_checksum(wl))
        for n in range(1, iters + 1):
            st = O.State(wl.poses0.astype(np.float64).copy(), wl.disps0.astype(np.float64).copy(),
                         wl.intr0.astype(np.float64).copy())
            res, rep = O.solve(st, prob, O.Options(iters=n, optimize_intrinsics=calib))
            out[f"poses_{n}"] = res.poses
            out[f"disps_{n}"] = res.disps.astype(np.float32)
            out[f"intr_{n}"] = res.intr
            out[f"energy_{n}"] = np.array(rep.energy_trace)
            out[f"trials_{n}"] = rep.trials
        np.savez_compressed(os.path.join(HERE, f"dba_{tag}.npz"), **out)
        print(f"{tag}: {len(wl.frames)} frames, {len(wl.ii)} edges, {H}x{W}, {iters} iterations, "
              f"{time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
