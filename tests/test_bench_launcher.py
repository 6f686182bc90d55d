"""bench.py --gpus N: the self-launch command and the per-rank edge shards (CPU, gloo)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_spawn_ranks_command(monkeypatch):
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench.spawn_ranks(types.SimpleNamespace(gpus=4)) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_ranks_shard_the_edges_by_source_frame(tmp_path):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    keyframes, world = 24, 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "tools", "rank_probe.py"), str(tmp_path), str(keyframes)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    outs = [json.load(open(tmp_path / f"rank{k}.json")) for k in range(world)]
    from paper_2411_17660_b200 import dba, scenes
    ii, _ = scenes.radius_edges(keyframes, scenes.CONFIGS[bench.CONFIG]["radius"])
    bounds = dba.partition(ii, keyframes, world)
    allloc = []
    for o in outs:
        k = o["rank"]
        assert o["world"] == world and o["local_rank"] == k
        assert (o["f0"], o["f1"]) == (int(bounds[k]), int(bounds[k + 1]))
        assert all(o["f0"] <= s < o["f1"] for s in o["src"])  # every local edge starts on the rank
        assert o["flow_rows"] == len(o["local"])
        allloc += o["local"]
    assert sorted(allloc) == list(range(len(ii)))  # a disjoint cover of the edge set
    assert np.all(np.diff(bounds) > 0)


def test_reference_arm_never_loads_the_library():
    """--impl reference runs the float64 CPU path only: no libdba_b200 and no CUDA library
    is mapped into the process (checked on a 10-keyframe graph)."""
    code = (
        "import sys, json; sys.argv=['bench.py','--impl','reference','--keyframes','10','--steps','1',"
        "'--warmup','0']; sys.path.insert(0, %r); import bench; bench.main(); "
        "maps=open('/proc/self/maps').read(); "
        "print(json.dumps({'dba': 'libdba_b200' in maps, 'cudart': 'libcudart' in maps or 'libcuda.so' in maps}))"
        % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, maps = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "port"
    assert not maps["dba"] and not maps["cudart"], maps
