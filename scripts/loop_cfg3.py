"""cfg3 (256^3 per rank) as a 4-rank loopback group on one GPU: a few solves, for ncu launch
lists of the reduced-phase and window kernels (measurement only)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2101_02286_b200 import ctri  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dims = (n * p, 256, 256)
dev = torch.device("cuda:0")
g = ctri.LoopbackGroup(dims, 0, p)
bs = [torch.rand((n, 256, 256), dtype=torch.float64, device=dev) for _ in range(p)]
xs = [torch.empty_like(t) for t in bs]
for _ in range(5):
    g.solve(bs, xs)
torch.cuda.synchronize()
print(g.stats(0))
