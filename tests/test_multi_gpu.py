"""NCCL path across real GPUs (torchrun, one rank per GPU); skipped with fewer than 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_nccl_partitions(world):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world),
           os.path.join(HERE, "mgpu_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULTS ")][-1]
    res = json.loads(line[len("RESULTS "):])
    if world <= 8:  # the opt-in runs with CTRI_FLAG_FUSED_REDUCED must have taken the fused
        # tile kernel (reduced_path 3); the default runs take the P2P kernel (reduced_path 1)
        assert any(v.get("path") == 3 for v in res.values()), res
    for k, v in res.items():
        assert v["err"] < 1e-12, (k, v)
        if "res" in v:
            assert v["res"] < 1e-13, (k, v)
            assert v["device_error"] == 0, (k, v)
