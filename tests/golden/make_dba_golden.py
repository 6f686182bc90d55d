"""Generate committed DBA golden fixtures from the float64 CPU oracle ("committed
.npz golden outputs from the oracle, per config and per iteration, then pin GPU parity").

    python tests/golden/make_dba_golden.py [TAG ...]

For each BASELINE config (C1 mono, C2 frontend window, C3 global backend, C4 depth prior,
C5 self-calibrating), at its own 48x64 resolution and for its full iteration budget, the
deterministic workload of ``paper_2411_17660_b200.scenes.make_workload`` is solved ONCE by
``oracle.dba.solve``; its ``snapshot`` hook records, after every accepted GN iteration n,
the state an ``iters=n`` call returns (poses and intrinsics float64, disparities through the
log-quantised codec of ``dba_codec.py``, 5e-7 relative), the energy trace and trial count.
Tags ending in ``n`` are the noisy variants (0.5 px Gaussian correspondence noise,
``providers.py:332-335``): their energy floor is the noise, so every LM decision of all
eight iterations is made by a real energy decrease, not by rounding.

The oracle's own float64 reproducibility floor is recorded next to each iteration: the
same solve is run a second time with equally valid float64 orderings (LAPACK LU instead
of Cholesky for the reduced solves, frame contributions accumulated in reverse order:
``Options(solver="lu", order="reverse")``).  On well-conditioned
pixels the two agree to ~1e-12; where a back-substitution cancels a large step almost
exactly (a noisy pixel driven towards zero disparity) the oracle disagrees WITH ITSELF by
up to ~1e-3 -- no float64 implementation can match it there to 1e-4.  Stored per
iteration: ``floor_idx_n`` / ``floor_rel_n`` (pixels where the two oracles differ by more
than 1e-6 relative), ``trials_lu_n`` and the LU run's iteration count ``iters_lu``.
``tests/test_dba_golden.py`` pins the oracle against C1 and compares the GPU path
against every fixture, every iteration.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import dba_codec  # noqa: E402
from oracle import dba as O  # noqa: E402
from paper_2411_17660_b200 import scenes  # noqa: E402

NOISE = 0.5
# tag -> (config, pixel noise)
FIXTURES = {
    "C1": ("C1", 0.0), "C2": ("C2", 0.0), "C3": ("C3", 0.0), "C4": ("C4", 0.0),
    "C5": ("C5", 0.0),
    "C1n": ("C1", NOISE), "C2n": ("C2", NOISE), "C3n": ("C3", NOISE), "C4n": ("C4", NOISE),
    "C5n": ("C5", NOISE),
}


def input_checksum(wl):
    h = np.float64(0.0)
    for a in (wl.poses0, wl.disps0, wl.flow, wl.intr0):
        x = np.asarray(a, np.float64).ravel()
        h += np.sum(x * (1.0 + np.arange(x.size) % 7))
    return float(h)


def make(tag):
    cfg, noise = FIXTURES[tag]
    t0 = time.time()
    wl = scenes.make_workload(cfg, noise=noise)
    H, W = wl.flow.shape[1:3]
    calib = bool(wl.optimize_intrinsics)
    prior = wl.prior is not None
    prob = O.Problem(ii=wl.ii, jj=wl.jj, flow=wl.flow, fixed=wl.fixed,
                     prior=wl.prior if prior else None, prior_mask=wl.prior_mask if prior else None)
    out = dict(config=cfg, noise=noise, height=H, width=W, keyframes=len(wl.frames),
               iters=wl.iters, calib=calib, prior=prior, checksum=input_checksum(wl))
    disps = []

    def snap(n, st, rep):
        out[f"poses_{n}"] = st.poses.copy()
        out[f"intr_{n}"] = st.intr.copy()
        out[f"energy_{n}"] = np.array(rep.energy_trace)
        out[f"trials_{n}"] = rep.trials
        disps.append(st.disps.copy())

    st = O.State(wl.poses0.astype(np.float64).copy(), wl.disps0.astype(np.float64).copy(),
                 wl.intr0.astype(np.float64).copy())
    _, rep = O.solve(st, prob, O.Options(iters=wl.iters, optimize_intrinsics=calib),
                     snapshot=snap)
    out["iters"] = rep.iterations

    def snap_lu(n, st2, rep2):  # the same solve, LU reduced solves: the oracle's own floor
        if n > len(disps):
            return
        rel = np.abs(st2.disps - disps[n - 1]) / disps[n - 1]
        idx = np.flatnonzero(rel > 1e-6)
        out[f"floor_idx_{n}"] = idx.astype(np.int32)
        out[f"floor_rel_{n}"] = rel.ravel()[idx]
        out[f"trials_lu_{n}"] = rep2.trials
        out[f"pose_lu_{n}"] = float(np.abs(st2.poses - out[f"poses_{n}"]).max())

    st = O.State(wl.poses0.astype(np.float64).copy(), wl.disps0.astype(np.float64).copy(),
                 wl.intr0.astype(np.float64).copy())
    _, rep_lu = O.solve(st, prob, O.Options(iters=wl.iters, optimize_intrinsics=calib, solver="lu",
                                                   order="reverse"),
                        snapshot=snap_lu)
    out["iters_lu"] = rep_lu.iterations
    out["initial_energy"] = rep.initial_energy
    for n, dl in enumerate(dba_codec.encode(wl.disps0, disps), 1):
        out[f"dq_{n}"] = dl
    np.savez_compressed(os.path.join(HERE, f"dba_{tag}.npz"), **out)
    floor = max([float(out[f"floor_rel_{n}"].max()) for n in range(1, rep_lu.iterations + 1)
                 if out.get(f"floor_rel_{n}") is not None and len(out[f"floor_rel_{n}"])] or [0.0])
    print(f"{tag}: {len(wl.frames)} frames, {len(wl.ii)} edges, {H}x{W}, {rep.iterations} "
          f"iterations, {rep.trials} trials (LU: {rep_lu.iterations} / {rep_lu.trials}), "
          f"max oracle self-disagreement {floor:.2e}, {time.time() - t0:.1f} s", flush=True)


def main():
    for tag in sys.argv[1:] or list(FIXTURES):
        make(tag)


if __name__ == "__main__":
    main()
