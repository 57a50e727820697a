"""Host-side multi-process logic on CPU with the gloo backend (world size 2): NCCL unique-id
broadcast, slab bounds, gather to rank 0 and max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2101_02286_b200 import dist as pdist
    uid = pdist.broadcast_unique_id(make_id=lambda: bytes(range(128)))
    lo, hi = pdist.slab_bounds(64, world, rank)
    local = torch.arange(lo, hi, dtype=torch.float64).reshape(hi - lo, 1, 1).repeat(1, 2, 3)
    g = pdist.gather_to_rank0(local, 0)
    mx = pdist.max_over_ranks(float(rank) + 0.5)
    if rank == 0:
        q.put((uid == bytes(range(128)), g[:, 0, 0].tolist() == list(range(64)), mx))
    else:
        q.put((uid == bytes(range(128)), g is None, mx))
    dist.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    outs = [q.get() for _ in range(2)]
    for ok_uid, ok_gather, mx in outs:
        assert ok_uid and ok_gather and mx == 1.5


def test_slab_bounds_errors():
    from paper_2101_02286_b200 import dist as pdist
    assert pdist.slab_bounds(8192, 8, 7) == (7168, 8192)
    with pytest.raises(ValueError):
        pdist.slab_bounds(10, 4, 0)
