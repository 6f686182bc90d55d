"""Per-source-line and per-opcode hot spots of one ncu --set full report (-lineinfo build).

  python profiles/tools/ncu_hot.py gpurun_out/pass_r02.ncu-rep [n_lines]
"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
f = None
cur = None
hdr = None
line_agg = collections.defaultdict(lambda: [0, 0])
op_agg = collections.defaultdict(lambda: [0, 0])
src = {}
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or hdr is None:
        continue
    if r[0].isdigit():
        cur = (f, int(r[0]))
        src[cur] = r[1].strip()[:80]
        continue
    if len(r) > 8 and cur is not None:
        try:
            e = int(r[7] or 0)
            smp = int(r[4] or 0)
        except ValueError:
            continue
        line_agg[cur][0] += e
        line_agg[cur][1] += smp
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
        if m:
            op_agg[m.group(2)][0] += e
            op_agg[m.group(2)][1] += smp
tot = sum(v[0] for v in line_agg.values()) or 1
tots = sum(v[1] for v in line_agg.values()) or 1
print(f"warp instructions {tot / 1e6:.2f} M, stall samples {tots}")
print("\n-- opcodes")
for k, v in sorted(op_agg.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{k:10s} {v[0] / 1e6:8.2f}M {v[0] / tot:6.3f}  samples {v[1] / tots:6.3f}")
print("\n-- source lines")
for k, v in sorted(line_agg.items(), key=lambda x: -x[1][0])[:nshow]:
    print(f"{k[0]}:{k[1]:4d} {v[0] / 1e6:7.2f}M {v[0] / tot:.3f} samples {v[1] / tots:.3f} | {src.get(k, '')}")
