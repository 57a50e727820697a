"""standalone NCCL send/recv ping-pong floor for one reduced-system plane (8m bytes,
m = 65536 -> 512 KiB) at partner distances 1, 2, 3 (torchrun, one rank per GPU).  Rank 0 pairs
with rank d; times 200 round trips with CUDA events; prints one JSON line."""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    res = {}
    for nbytes in (8 * 65536, 8 * 262144, 8):
        buf = torch.ones(nbytes // 8, dtype=torch.float64, device=dev)
        for d in range(1, world):
            dist.barrier()
            reps = 200
            if rank in (0, d):
                peer = d if rank == 0 else 0
                for _ in range(10):
                    if rank == 0:
                        dist.send(buf, peer); dist.recv(buf, peer)
                    else:
                        dist.recv(buf, peer); dist.send(buf, peer)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    if rank == 0:
                        dist.send(buf, peer); dist.recv(buf, peer)
                    else:
                        dist.recv(buf, peer); dist.send(buf, peer)
                e1.record()
                torch.cuda.synchronize()
                if rank == 0:
                    rt = e0.elapsed_time(e1) * 1e3 / reps
                    res[f"{nbytes}B_distance{d}"] = {"round_trip_us": round(rt, 2), "one_way_us": round(rt / 2, 2),
                                                     "GBps_one_way": round(nbytes / (rt / 2 * 1e-6) / 1e9, 1)}
            dist.barrier()
    if rank == 0:
        print(json.dumps({"what": "NCCL send/recv ping-pong (host-issued, torch.distributed)", "world": world,
                          "results": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
