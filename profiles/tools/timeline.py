import sys, os
sys.path.insert(0, '/root/repo')
os.environ['DBA_TIMELINE'] = '1'
import torch, bench
from paper_2411_17660_b200 import dba
inp = bench.build_inputs(300, 0, 1)
s = dba.DBASolver(inp['ii'], inp['jj'], 300, 48, 64, inp['fixed'])
dev = torch.device('cuda')
P = torch.as_tensor(inp['poses0'], device=dev); D = torch.as_tensor(inp['disps0'], device=dev)
K = torch.as_tensor(inp['intr0'], device=dev); F = torch.as_tensor(inp['flow'], device=dev)
for _ in range(2): s.solve(P, D, K, F, iters=8)
torch.cuda.synchronize()
s.set_profiling(True)
print('--- one solve (8 iterations)', file=sys.stderr)
s.solve(P, D, K, F, iters=8)
