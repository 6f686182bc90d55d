"""Per-CTA load balance of pass_kernel on the bench workload (noisy C3).

Builds a diagnostic variant of the library with -DDBA_PASS_TIMING (per-CTA globaltimer
stamps at entry and when the last product / linearisation warp finishes), runs one
linearisation (build_system) after warm-up, and prints the spread of CTA durations next
to each CTA's share of the plan's contiguous (frame, tile) split.

    python profiles/tools/pass_balance.py [repeats]
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
LIB = os.environ.get("DBA_TIMING_LIB", "/tmp/libdba_b200_timing.so")


def build_variant():
    from paper_2411_17660_b200 import build as B
    src = B.SRC
    cmd = [B.nvcc_path(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-DDBA_PASS_TIMING", "-Xcompiler", "-fPIC",
           "-shared", "-o", LIB, str(src / "dba_host.cu"), str(src / "dba_ingest.cu"), str(src / "dba_graph.cu"),
           str(src / "dba_prgbd.cu"), str(src / "dba_provider.cu"), "-ldl"]
    subprocess.run(cmd, check=True)


def tile_cost(k, calib=False):
    mpad = (6 * max(k, 1) + (4 if calib else 0) + 2 + 15) & ~15
    np_ = mpad >> 4
    return 2880 + 100 * k + 95 * (2 * np_ * (np_ - 1) + 3 * np_)


def split(csr_counts, n_tiles, G):
    """The plan's weighted contiguous split (dba_host.cu, fitted tile cost)."""
    tot = sum(tile_cost(k) * n_tiles for k in csr_counts)
    cum, cur_cta, cur_fl = 0, -1, -1
    segs = [[] for _ in range(G)]
    for fl, k in enumerate(csr_counts):
        c = tile_cost(k)
        for t in range(n_tiles):
            cta = min(G - 1, ((2 * cum + c) * G) // (2 * max(tot, 1)))
            cta = max(cta, max(cur_cta, 0))
            if cta != cur_cta or fl != cur_fl:
                segs[cta].append([fl, t, t + 1])
                cur_cta, cur_fl = cta, fl
            else:
                segs[cta][-1][2] = t + 1
            cum += c
    return segs


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    if not os.path.exists(LIB):
        build_variant()
    os.environ["DBA_B200_LIB"] = LIB
    import torch
    import bench
    from paper_2411_17660_b200 import _lib, dba
    lib = _lib.load()
    lib.dba_debug_pass_times.restype = ctypes.c_int
    lib.dba_debug_pass_times.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    inp = bench.build_inputs(300, 0, 1)
    s = dba.DBASolver(inp["ii"], inp["jj"], 300, 48, 64, inp["fixed"])
    dev = torch.device("cuda")
    P = torch.as_tensor(inp["poses0"], device=dev)
    D = torch.as_tensor(inp["disps0"], device=dev)
    K = torch.as_tensor(inp["intr0"], device=dev)
    F = torch.as_tensor(inp["flow"], device=dev)
    G = int(s.info.n_split)
    buf = (ctypes.c_ulonglong * (4 * 1024))()
    counts = np.bincount(np.asarray(inp["ii"]), minlength=300)
    segs = split([int(c) for c in counts if c > 0], (48 * 64 + 127) // 128, G)
    durs = []
    for r in range(reps + 1):
        lib.dba_debug_pass_times(None, 0)
        s.build_system(P, D, K, F)
        torch.cuda.synchronize()
        lib.dba_debug_pass_times(buf, 4 * G)
        t = np.array(buf[:4 * G], dtype=np.float64).reshape(G, 4)
        sm = t[:, 3].astype(int)
        if r == 0:
            continue  # warm-up
        t0 = t[:, 0].min()
        durs.append(np.stack([t[:, 0] - t0, t[:, 1] - t0, t[:, 2] - t0], 1) / 1e3)  # us
    d = np.median(np.stack(durs), 0)
    end = np.maximum(d[:, 1], d[:, 2])
    print(f"CTAs {G}: kernel span {end.max():.1f} us; CTA end mean {end.mean():.1f} min {end.min():.1f} "
          f"max {end.max():.1f}; start spread {d[:, 0].max():.1f} us")
    print(f"  product-warps end mean {d[:, 1].mean():.1f}  linearisation end mean {d[:, 2].mean():.1f}")
    tiles = np.array([sum(b - a for _, a, b in sg) for sg in segs])
    nseg = np.array([len(sg) for sg in segs])
    for ns in sorted(set(nseg)):
        m = nseg == ns
        print(f"  CTAs with {ns} segments: {m.sum():3d}, tiles {tiles[m].mean():.1f}, end mean {end[m].mean():.1f} "
              f"max {end[m].max():.1f}")
    order = np.argsort(-end)
    print("  slowest CTAs (cta: end us, start us, segments [frame, t0, t1]):")
    for g in order[:8]:
        print(f"   {g:3d}: {end[g]:.1f} {d[g, 0]:.1f} {segs[g]}")
    print("  fastest:")
    for g in order[-4:]:
        print(f"   {g:3d}: {end[g]:.1f} {d[g, 0]:.1f} {segs[g]}")
    out = os.environ.get("PASS_BALANCE_JSON")
    if out:
        import json
        json.dump({"end": end.tolist(), "start": d[:, 0].tolist(), "sm": sm.tolist(), "segs": segs}, open(out, "w"))


if __name__ == "__main__":
    main()
