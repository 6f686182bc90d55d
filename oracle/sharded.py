"""Edge-sharded DBA step on CPU — TEST INFRASTRUCTURE ONLY.

The multi-GPU decomposition of libdba_b200: source frames
are partitioned into contiguous ranges (``dba_partition``: balanced out-degree + 1
weight); every rank linearises only the edges whose source frame it owns (all of
that frame's disparity terms are local), the packed reduced systems and energies
are SUMMED across ranks (one all-reduce), every rank solves the identical system,
and back-substitutes its own frames.  ``allreduce`` is injected so the same code
runs under torch.distributed (gloo) in tests/test_sharded_oracle.py.
"""

from __future__ import annotations

import numpy as np

from . import dba as O


def partition(ii, n_frames, nranks):
    """Restatement of dba_partition (paper_2411_17660_b200/csrc/dba_host.cu)."""
    w = np.ones(n_frames, dtype=np.int64)
    np.add.at(w, np.asarray(ii, dtype=np.int64), 1)
    pre = np.concatenate([[0], np.cumsum(w)])
    b = [0]
    for r in range(1, nranks):
        f = int(np.argmax(pre * nranks >= r * pre[-1]))
        b.append(max(f, b[-1]))
    b.append(n_frames)
    return np.array(b)


def sharded_step(state, prob, opts, rank, nranks, allreduce, lam):
    """One damped GN step (linearise, all-reduce, solve, back-substitute) on this
    rank's frames.  Returns (new disparities of the local frames, new poses, the
    summed reduced system S, y and energy)."""
    N = state.poses.shape[0]
    b = partition(prob.ii, N, nranks)
    frames = list(range(int(b[rank]), int(b[rank + 1])))
    sysm = O.linearize(state, prob, opts, frames=frames)
    packed = np.concatenate([sysm.S.ravel(), sysm.y, [sysm.energy]])
    packed = allreduce(packed)
    n = sysm.S.shape[0]
    S = packed[:n * n].reshape(n, n)
    y = packed[n * n:n * n + n]
    energy = float(packed[-1])
    full = O.System(S, y, energy, sysm.edge_energy, sysm.edge_finite, sysm.C, sysm.gd)
    Sr, yr, _ = O.reduced(full, prob, opts)
    delta, _ = O.solve_reduced(Sr, yr, lam)
    dxi, dth = O.split_step(delta, prob.fixed, opts.optimize_intrinsics)
    dxi = O.clamp_tangents(dxi, opts.tangent_max)
    new = O.backsub_and_retract(state, prob, opts, dxi, dth, frames=frames)
    return new.disps[frames], new.poses, S, y, energy, frames
