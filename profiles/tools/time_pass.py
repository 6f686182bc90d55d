import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2411_17660_b200 import dba
inp = bench.build_inputs(300, 0, 1)
s = dba.DBASolver(inp['ii'], inp['jj'], 300, 48, 64, inp['fixed'])
dev = torch.device('cuda')
P = torch.as_tensor(inp['poses0'], device=dev); D = torch.as_tensor(inp['disps0'], device=dev)
K = torch.as_tensor(inp['intr0'], device=dev); F = torch.as_tensor(inp['flow'], device=dev)
for _ in range(2): s.build_system(P, D, K, F)
s.set_profiling(True); s.stats(reset=True)
for _ in range(5): s.build_system(P, D, K, F)
st = s.stats(reset=True)
print(os.environ.get('DBA_B200_LIB', 'default'), 'init-pass ms', st['pass_ms'] / st['pass_launches'])
try:
    for _ in range(3): s.debug_trial(P, D, K, F)
    st = s.stats(reset=True)
    print('   trial-pass ms (2 passes/call avg)', st['pass_ms'] / max(st['pass_launches'], 1), 'solve', st['solve_ms'] / max(st['solve_launches'], 1))
except Exception as e:
    print('   trial failed', e)
