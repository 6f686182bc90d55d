"""Launched by tests/test_bench_launcher.py under torch.distributed.run (gloo, CPU): each rank
builds its bench inputs exactly as bench.py does and reports its shard."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2411_17660_b200 import dba  # noqa: E402

rank, local_rank, world = bench.dist_env()
dist.init_process_group("gloo")
inp = bench.build_inputs(int(sys.argv[2]), rank, world, dba.partition, noise=0.5)
out = dict(rank=rank, local_rank=local_rank, world=world, f0=inp["f0"], f1=inp["f1"],
           local=[int(e) for e in inp["local"]], n_edges=len(inp["ii"]),
           src=[int(inp["ii"][e]) for e in inp["local"]], flow_rows=int(inp["flow"].shape[0]))
with open(os.path.join(sys.argv[1], f"rank{rank}.json"), "w") as fh:
    json.dump(out, fh)
dist.barrier()
dist.destroy_process_group()
