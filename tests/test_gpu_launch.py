"""The driver's launch paths of bench.py on a GPU box: one rank under
torch.distributed.run (NCCL process group, solver on cuda:LOCAL_RANK), and --
where the box has them -- two ranks on two devices with the config-3 batch
sharded between them (no collective on the solve path)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _line(out):
    return json.loads([l for l in out.strip().splitlines() if l.startswith("{")][-1])


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


@pytest.mark.gpu
def test_torchrun_one_rank():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29631", BENCH, "--gpus", "1",
           "--workload", "c0", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    j = _line(out.stdout)
    assert j["n_gpus"] == 1 and j["value"] > 0 and j["gpu_launches"] > 0
    assert j["run_info"]["devices"] == [0]
    assert j["e2e"]["h2d_bytes_per_step"] > 0 and j["roofline"]["frac"] > 0


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
def test_two_ranks_two_devices():
    """`bench.py --gpus 2` spawns one rank per GPU; each solver runs on its own
    device and owns half of the 256 sections."""
    cmd = [sys.executable, BENCH, "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--no-extras"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    j = _line(out.stdout)
    assert j["n_gpus"] == 2 and j["run_info"]["devices"] == [0, 1]
    assert j["run_info"]["sections_per_rank"] == 128
