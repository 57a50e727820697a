"""Memory ceiling of the tile kernel's access pattern: with CTRI_TILE_COPY_ONLY=1 the kernel runs
x = b through the same TMA ring / store path (no solve); compared with torch's contiguous copy_."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2101_02286_b200 import ctri  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dims, sd = workloads.config(cfg)
dev = torch.device("cuda:0")
b = workloads.device_uniform(dims, 2, dev)
x = torch.empty_like(b)
plan = ctri.Plan(dims, sd)


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ms = timeit(lambda: plan.solve(b, x))
ms_copy = timeit(lambda: x.copy_(b))
nbytes = 16 * b.numel()
st = plan.stats()
print(json.dumps({"cfg": cfg, "variant": st["tile_variant"], "K": st["rows_per_thread"],
                  "G": st["cluster_size"], "copy_only": bool(os.environ.get("CTRI_TILE_COPY_ONLY")),
                  "tile_ms": ms, "tile_GBps": nbytes / ms / 1e6,
                  "torch_copy_ms": ms_copy, "torch_copy_GBps": nbytes / ms_copy / 1e6}))
