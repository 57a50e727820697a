"""torchrun worker for tests/test_multi_gpu.py: the NCCL path of ctri_solve / ctri_deriv on
p = WORLD_SIZE GPUs, gathered to rank 0 and compared with the CPU oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np
import torch
import torch.distributed as dist

import oracle
import workloads
from helpers import rel_err, residual
from paper_2101_02286_b200 import (CTRI_FLAG_DERIV, CTRI_FLAG_NCCL_ROUNDS, CTRI_FLAG_TIMING,
                                   CTRI_FLAG_FUSED_REDUCED)
from paper_2101_02286_b200 import dist as pdist


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    results = {}
    cases = [((64 * world, 8, 16), 0, (1 / 3, 1.0, 1 / 3), True),
             ((256 * world, 4, 32), 0, (0.45, 1.0, 0.45), True),
             ((256 * world, 2, 48), 0, (0.2, 1.1, 0.4), True),
             ((8, 128 * world, 32), 1, (1 / 3, 1.0, 1 / 3), True),
             ((4, 6, 64 * world), 2, (1 / 3, 1.0, 1 / 3), True),
             ((96 * world, 3, 16), 0, (0.2, 1.1, 0.4), False),
             # slabs the fused tile kernel takes (window rows stashed across a 4/8-CTA cluster)
             ((1024 * world, 2, 64), 0, (1 / 3, 1.0, 1 / 3), True),
             ((2048 * world, 1, 40), 0, (0.45, 1.0, 0.45), True),   # ragged batch, wide window
             ((1024 * world, 2, 64), 0, (0.2, 1.1, 0.4), False),
             ((4, 1024 * world, 64), 1, (1 / 3, 1.0, 1 / 3), True)]
    pow2 = (world & (world - 1)) == 0
    runs = [(c, fl) for c in cases for fl in (0, CTRI_FLAG_FUSED_REDUCED, CTRI_FLAG_NCCL_ROUNDS)
            if pow2 or fl != CTRI_FLAG_NCCL_ROUNDS or not c[3]]  # cyclic non-power-of-two: P2P only
    for idx, ((dims, sd, bands, cyc), fl) in enumerate(runs):
        b = workloads.uniform(dims, 6 + idx)
        plan = pdist.plan_from_process_group(dims, sd, bands, cyc, flags=CTRI_FLAG_TIMING | fl)
        bl = torch.from_numpy(workloads.slab(b, sd, world, rank)).to(dev)
        xl = torch.empty_like(bl)
        plan.solve(bl, xl)
        torch.cuda.synchronize()
        st = plan.stats()
        x = pdist.gather_to_rank0(xl, sd)
        plan.close()
        if rank == 0:
            xn = x.cpu().numpy()
            ref = oracle.cyclic_solve(b, sd, bands) if cyc else oracle.acyclic_solve(b, sd, bands)
            results[f"case{idx}"] = {"err": rel_err(xn, ref, sd),
                                     "res": residual(xn, b, sd, bands, cyc),
                                     "stages": st["pcr_stages"], "sends": st["sends_per_solve"],
                                     "kernel": st["local_kernel"], "path": st["reduced_path"],
                                     "device_error": st["device_error"]}
    # the default P2P path captured in one CUDA graph (programmatic dependent launches,
    # device-resident epochs), replayed three times; stats read the captured phase events
    dims = (1024 * world, 2, 64)
    b = workloads.uniform(dims, 99)
    plan = pdist.plan_from_process_group(dims, 0, flags=CTRI_FLAG_TIMING)
    bl = torch.from_numpy(workloads.slab(b, 0, world, rank)).to(dev)
    xl = torch.empty_like(bl)
    plan.solve(bl, xl)  # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.solve(bl, xl)
    for _ in range(3):
        xl.zero_()
        g.replay()
    torch.cuda.synchronize()
    st = plan.stats()
    x = pdist.gather_to_rank0(xl, 0)
    plan.close()
    if rank == 0:
        results["graph"] = {"err": rel_err(x.cpu().numpy(), oracle.cyclic_solve(b, 0), 0),
                            "p2p_us": st["t_reduced_kernel_us"], "window_us": st["t_window_us"],
                            "steps": st["p2p_steps"]}
        assert st["t_reduced_kernel_us"] > 0 and st["t_window_us"] > 0, st
    # compact derivative over NCCL (halo exchange)
    dims = (128 * world, 4, 16)
    f = workloads.cfg5_field(dims, 0, 5, kappas=(1, 5, 13))
    plan = pdist.plan_from_process_group(dims, 0, flags=CTRI_FLAG_DERIV)
    fl = torch.from_numpy(workloads.slab(f, 0, world, rank)).to(dev)
    dl = torch.empty_like(fl)
    plan.deriv(fl, dl)
    torch.cuda.synchronize()
    d = pdist.gather_to_rank0(dl, 0)
    plan.close()
    if rank == 0:
        results["deriv"] = {"err": rel_err(d.cpu().numpy(), oracle.deriv(f, 0), 0)}
    # pentadiagonal (r = 2) partition method over real GPUs (IPC all-gather)
    pb = (-0.07, 0.21, 1.3, -0.33, 0.11)
    pdims = (16 * world, 3, 40)
    b = workloads.uniform(pdims, 95)
    plan = pdist.plan_from_process_group(pdims, 0, pb, True)
    bl = torch.from_numpy(workloads.slab(b, 0, world, rank)).to(dev)
    xl = torch.empty_like(bl)
    plan.solve(bl, xl)
    torch.cuda.synchronize()
    x = pdist.gather_to_rank0(xl, 0)
    plan.close()
    if rank == 0:
        results["penta"] = {"err": rel_err(x.cpu().numpy(), oracle.penta_solve(b, 0, pb, True), 0)}
    # pentadiagonal with the on-chip local solve (1024-row slabs) and the 2x2-block schedule
    # (block detach / reattach at 3 GPUs), Lele's tenth-order LHS
    pb2 = (1 / 20, 1 / 2, 1.0, 1 / 2, 1 / 20)
    pdims = (1024 * world, 1, 64)
    b = workloads.uniform(pdims, 96)
    plan = pdist.plan_from_process_group(pdims, 0, pb2, True)
    bl = torch.from_numpy(workloads.slab(b, 0, world, rank)).to(dev)
    xl = torch.empty_like(bl)
    plan.solve(bl, xl)
    torch.cuda.synchronize()
    st = plan.stats()
    x = pdist.gather_to_rank0(xl, 0)
    plan.close()
    if rank == 0:
        results["penta_chip"] = {"err": rel_err(x.cpu().numpy(), oracle.penta_solve(b, 0, pb2, True), 0),
                                 "kernel": st["local_kernel"], "path": st["reduced_path"],
                                 "detached": st["detached_rows"]}
        assert st["local_kernel"] == 4 and st["reduced_path"] == 1, st
    # pentadiagonal with 2048-row slabs: two on-chip partitions per GPU as virtual rows of the
    # 2x2-block reduced system (2 * world block rows; rows of one GPU through its own mailbox)
    pdims = (2048 * world, 1, 64)
    b = workloads.uniform(pdims, 97)
    plan = pdist.plan_from_process_group(pdims, 0, pb2, True)
    bl = torch.from_numpy(workloads.slab(b, 0, world, rank)).to(dev)
    xl = torch.empty_like(bl)
    plan.solve(bl, xl)
    torch.cuda.synchronize()
    st = plan.stats()
    x = pdist.gather_to_rank0(xl, 0)
    plan.close()
    if rank == 0:
        results["penta_vrows"] = {"err": rel_err(x.cpu().numpy(), oracle.penta_solve(b, 0, pb2, True), 0),
                                  "kernel": st["local_kernel"], "path": st["reduced_path"],
                                  "rows": st["reduced_rows"]}
        assert st["local_kernel"] == 4 and st["vparts"] == 2 and st["reduced_rows"] == 2 * world, st
    # staggered sixth-order interpolation through ctri_compact_apply
    from paper_2101_02286_b200 import ctri
    plan = pdist.plan_from_process_group(dims, 0, ctri.staggered_interp_bands(), True, flags=CTRI_FLAG_DERIV)
    plan.compact_apply(ctri.staggered_interp_coef(), fl, dl)
    torch.cuda.synchronize()
    d = pdist.gather_to_rank0(dl, 0)
    plan.close()
    if rank == 0:
        ref = oracle.compact_apply(f, 0, oracle.staggered_interp_coef(), oracle_bands_interp())
        results["sinterp"] = {"err": rel_err(d.cpu().numpy(), ref, 0)}
        print("RESULTS " + json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def oracle_bands_interp():
    return (oracle.STAGGERED_INTERP_ALPHA, 1.0, oracle.STAGGERED_INTERP_ALPHA)


if __name__ == "__main__":
    main()
