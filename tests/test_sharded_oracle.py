"""Multi-rank decomposition on CPU (gloo, world_size 2): the edge-sharded step
(oracle/sharded.py — the algorithm libdba_b200 runs with one NCCL all-reduce per GN
trial) equals the unsharded oracle step, and the frame partition matches the
library's dba_partition."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import dba as O
    from oracle import sharded
    from tests.helpers import oracle_problem, oracle_state, small_workload
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = small_workload("C1", height=16, width=24)
    st = oracle_state(wl)
    prob = oracle_problem(wl)
    opts = O.Options()

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    d_loc, poses, S, y, e, frames = sharded.sharded_step(st, prob, opts, rank, world, allreduce, 1e-4)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), d=d_loc, poses=poses, S=S, y=y, e=e,
             frames=np.array(frames))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_equals_unsharded(tmp_path):
    from oracle import dba as O
    from tests.helpers import oracle_problem, oracle_state, small_workload
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    wl = small_workload("C1", height=16, width=24)
    st = oracle_state(wl)
    prob = oracle_problem(wl)
    opts = O.Options()
    full = O.linearize(st, prob, opts)
    Sr, yr, _ = O.reduced(full, prob, opts)
    delta, _ = O.solve_reduced(Sr, yr, 1e-4)
    dxi, dth = O.split_step(delta, prob.fixed, False)
    ref = O.backsub_and_retract(st, prob, opts, O.clamp_tangents(dxi, 1.0), dth)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for o in outs:
        assert np.allclose(o["S"], full.S, rtol=1e-12, atol=1e-9 * np.abs(full.S).max())
        assert np.allclose(o["y"], full.y, rtol=1e-12, atol=1e-9 * np.abs(full.y).max())
        assert float(o["e"]) == pytest.approx(full.energy, rel=1e-12)
        assert np.allclose(o["poses"], ref.poses, atol=1e-12)
    frames = np.concatenate([o["frames"] for o in outs])
    assert np.array_equal(np.sort(frames), np.arange(len(wl.frames)))  # partition covers all
    d = np.concatenate([o["d"] for o in outs])
    assert np.allclose(d, ref.disps[frames], rtol=1e-12)
    # ranks ran identical solves: bit-identical poses
    assert np.array_equal(outs[0]["poses"], outs[1]["poses"])


def test_oracle_partition_matches_library():
    from oracle import sharded
    from paper_2411_17660_b200 import dba, scenes
    for n, r, R in ((300, 5, 8), (25, 3, 2), (9, 1, 4)):
        ii, _ = scenes.radius_edges(n, r)
        assert np.array_equal(sharded.partition(ii, n, R), dba.partition(ii, n, R))
