"""Multi-GPU: the ghost exchange (one-sided NVLink puts, and NCCL send/recv)
reproduces single-rank results bitwise (runs tests/mp_fmm_run.py under
torchrun on 2 GPUs; skipped with < 2 GPUs)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("transport,port,xmode", [("puts", 29533, "1"), ("nccl", 29535, "1"), ("puts", 29537, "0")])
def test_two_rank_bitwise(gpu, transport, port, xmode):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OCTO_XCHG=transport, OCTO_XMODE=xmode)   # xmode 0: exchange overlapped, split rounds
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tests", "mp_fmm_run.py")], capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
