import sys
sys.path.insert(0, '/root/repo')
import torch
import bench
from paper_2411_17660_b200 import dba
inp = bench.build_inputs(300, 0, 1)
s = dba.DBASolver(inp['ii'], inp['jj'], 300, 48, 64, inp['fixed'])
dev = torch.device('cuda')
P = torch.as_tensor(inp['poses0'], device=dev); D = torch.as_tensor(inp['disps0'], device=dev)
K = torch.as_tensor(inp['intr0'], device=dev); F = torch.as_tensor(inp['flow'], device=dev)
_, _, _, rep = s.solve(P, D, K, F, iters=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
torch.cuda.synchronize()
print('trials', rep.trials, 'iters', rep.iterations_run)
