"""Multi-GPU: the distributed Q3 shuffle join over NCCL, one process per GPU
(torchrun), vs the oracle.  Needs >= 2 GPUs (gpurun --gpus 2/4)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("mode", ["lip", "nolip", "engine", "fused", "fused_nolip"])
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_q3_nccl(world, mode):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), os.path.join(ROOT, "tests", "mgpu_q3.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, TQ_SF="0.1", TQ_LIP="1" if mode in ("lip", "fused") else "0",
                                TQ_ENGINE="1" if mode == "engine" else "0",
                                TQ_FUSED="1" if mode.startswith("fused") else "0"))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "mgpu q3 ok" in r.stdout


@pytest.mark.parametrize("mode", ["validity", "engine", "utf8"])
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_ops(world, mode):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tests", "mgpu_ops.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, TQ_MODE=mode))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "mgpu ops ok" in r.stdout
