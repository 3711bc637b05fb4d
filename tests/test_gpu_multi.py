"""Multi-rank ghost exchange: several
ranks reproduce single-rank results bitwise over several steps with new
densities each step (runs tests/mp_fmm_run.py under torchrun).

* `test_two_ranks_one_gpu_bitwise` runs on ANY GPU box: two processes share
  cuda:0, the one-sided NVLink-put exchange (CUDA IPC arenas, release/acquire
  epoch flags) is bootstrapped through a torch gloo allgather
  (OCTO_EXTERNAL_BOOTSTRAP), so no NCCL communicator is needed.
* `test_two_rank_bitwise` uses one process per GPU and the library's own NCCL
  communicator (both transports); it needs 2 GPUs.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(nproc, port, env_extra, timeout=1500):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "mp_fmm_run.py")], capture_output=True, text=True,
                       timeout=timeout, env=env)
    return r


def test_two_ranks_one_gpu_bitwise(gpu):
    r = _run(2, 29531, {"OCTO_MP_BOOT": "gloo", "OCTO_XCHG": "puts", "OCTO_MP_STEPS": "4",
                        "OCTO_MP_TREES": "c3,amr,v1309-13"})
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("transport,port,xmode", [("puts", 29533, "1"), ("nccl", 29535, "1"), ("puts", 29537, "0")])
def test_two_rank_bitwise(gpu, transport, port, xmode):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (the 1-GPU variant is test_two_ranks_one_gpu_bitwise)")
    # xmode 0: exchange overlapped with interior nodes, split rounds
    r = _run(2, port, {"OCTO_XCHG": transport, "OCTO_XMODE": xmode})
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
