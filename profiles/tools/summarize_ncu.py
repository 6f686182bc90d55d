"""Summarise the round's ncu captures into profiles/ (tracked)."""
import csv, collections, json, subprocess, sys, os
out_dir = sys.argv[1]
tag = sys.argv[2]
g = '/root/repo/gpurun_out'
lines = []
# launch list
rows = list(csv.reader(open(f'{g}/launches.csv')))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0, 0, 0.0])
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] != 'gpu__time_duration.sum': continue
        v = float(d['Metric Value'].replace(',', ''))
        v *= {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(d['Metric Unit'], 1.0)
        name = d['Kernel Name'].split('(')[0]
        agg[name][0] += 1; agg[name][1] += v
        if v > 12.0: agg[name][2] += 1; agg[name][3] += v  # ran (gated-off launches return in a few us)
tot = sum(v[1] for v in agg.values())
lines.append(f'## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n')
lines.append('Gated kernels (energy/pass/assemble/gather of candidates and linearisations the LM decision '
             'rules out) return at entry; "ran" counts launches longer than 12 us.\n')
lines.append('| kernel | launches | total us | avg us | ran | avg us (ran) | share |\n|---|---|---|---|---|---|---|')
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    ran = f'{v[3]/v[2]:.2f}' if v[2] else '-'
    lines.append(f'| `{k}` | {v[0]} | {v[1]:.1f} | {v[1]/v[0]:.2f} | {v[2]} | {ran} | {v[1]/tot:.3f} |')
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_metrics import WANT as want  # noqa: E402
res = {}
for rep in ('pass', 'solve', 'energy'):
    raw = subprocess.run(['ncu', '-i', f'{g}/{rep}_{tag}.ncu-rep', '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    m = {}
    for w in want:
        if w in h:
            i = h.index(w); m[w] = (v[i], u[i])
    stalls = {}
    for i, n in enumerate(h):
        if 'pcsamp_warps_issue_stalled' in n and 'not_issued' not in n:
            try:
                if float(v[i]) > 0: stalls[n.replace('smsp__pcsamp_warps_issue_stalled_', '')] = int(float(v[i]))
            except ValueError: pass
    res[rep] = (m, stalls)
    lines.append(f'\n## `{rep}_kernel` (ncu --set full --clock-control none, one launch)\n')
    lines.append('| metric | value | unit |\n|---|---|---|')
    for k, (a, b) in m.items():
        lines.append(f'| {k} | {a} | {b} |')
    top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
    lines.append('\nTop warp-stall samples: ' + ', '.join(f'{k} {v}' for k, v in top))
open(os.path.join(out_dir, f'{tag}_ncu_summary.md'), 'w').write('\n'.join(lines) + '\n')
pm = res['pass'][0]
def num(k):
    a, b = pm[k]; x = float(a.replace(',', ''))
    return x * {'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'byte': 1.0}.get(b, 1.0)
json.dump({'kernel': 'dba::pass_kernel', 'round': tag, 'dram_bytes_per_launch': num('dram__bytes_read.sum') + num('dram__bytes_write.sum'),
           'dram_read': num('dram__bytes_read.sum'), 'dram_write': num('dram__bytes_write.sum'),
           'duration_us': float(pm['gpu__time_duration.sum'][0]) * (1e-3 if pm['gpu__time_duration.sum'][1] == 'nsecond' else 1.0),
           'source': f'profiles/{tag}_ncu_summary.md'}, open(os.path.join(out_dir, 'pass_kernel_ncu.json'), 'w'), indent=1)
print(open(os.path.join(out_dir, f'{tag}_ncu_summary.md')).read())
