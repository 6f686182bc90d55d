"""Headline metrics + stall breakdown of ncu --set full reports.

  python profiles/tools/ncu_metrics.py gpurun_out/pass_r02.ncu-rep [...]
"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    m = {w: (v[h.index(w)], u[h.index(w)]) for w in WANT if w in h}
    st = {}
    for i, n in enumerate(h):
        if "pcsamp_warps_issue_stalled" in n and "not_issued" not in n:
            try:
                if float(v[i]) > 0:
                    st[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v[i]))
            except ValueError:
                pass
    return m, st


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        m, st = metrics(rep)
        print(f"== {rep}")
        for k, (a, b) in m.items():
            print(f"  {k:75s} {a} {b}")
        tot = sum(st.values()) or 1
        print("  stalls: " + ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
