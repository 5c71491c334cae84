"""Multi-GPU parity through the C-ABI on the GPUs of this box (skipped with
fewer than two): scripts/mgpu_check.py under torchrun -- every leaf op with
an NCCL communicator against the CPU restatement, placed / host-staged /
repartitioned pieces, SpAdd3 row blocks, and uneven colour blocks
(spd_context_set_colour_blocks) with placement following them."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
def test_two_gpu_check():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "scripts", "mgpu_check.py")],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "MGPU_RESULT PASS" in r.stdout, r.stdout[-4000:] + r.stderr[-3000:]
    assert "blocks" in r.stdout and "MISMATCH" not in r.stdout


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
def test_abort_unblocks_a_waiting_rank():
    """spd_context_abort: a rank waiting in the boundary all-gather for a
    peer that never joins returns an error once its communicator is aborted
    (what execute_gpu does for the other GPUs when one of them fails)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "abort_check.py")],
                       capture_output=True, text=True, timeout=180)
    assert "ABORT_RESULT PASS" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
