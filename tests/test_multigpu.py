"""One rank per GPU over NVLink/NVSwitch: runs tests/mp_check.py under torchrun
on every available GPU (2..8).  Skipped on a single-GPU box; the same protocol
runs on one GPU in tests/test_gpu_engine.py (emulated world)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import need_gpus

pytestmark = pytest.mark.multigpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_process_world_parity():
    need_gpus(2)
    import torch
    p = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "tests", "mp_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = res.stdout
    start = out.find("{")
    assert start >= 0, res.stdout[-3000:] + res.stderr[-3000:]
    summary = json.loads(out[start:out.rfind("}") + 1])
    assert res.returncode == 0 and summary["ok"], json.dumps(summary, indent=1)


def test_process_world_p8_two_ranks_per_gpu():
    """P=8 geometry (8 KiB chunks, 2 TMA stages, rs_fixed<8>) across processes
    on a 4-GPU box: two ranks (and engines) per GPU.  Data-path parity only --
    the engines of two processes time-slice a GPU without MPS, so arrival-order
    checks are skipped.  On an 8-GPU box the test above already runs P=8."""
    need_gpus(4)
    import torch
    if torch.cuda.device_count() >= 8:
        pytest.skip("P=8 runs one rank per GPU in test_process_world_parity")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", str(30500 + os.getpid() % 1000),
           os.path.join(ROOT, "tests", "mp_check.py")]
    env = dict(os.environ, EC_RANKS_PER_GPU="2")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    out = res.stdout
    start = out.find("{")
    assert start >= 0, res.stdout[-3000:] + res.stderr[-3000:]
    summary = json.loads(out[start:out.rfind("}") + 1])
    assert res.returncode == 0 and summary["ok"], json.dumps(summary, indent=1)
