"""Multi-GPU parity: R = 2 / 4 ranks (torchrun, NCCL) bit-identical to R = 1 (tests/mgpu_worker.py).
Skipped when the box has fewer GPUs than ranks."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ranks,n,xi,peer", [(2, 60000, 1e-3, "1"), (2, 120000, 3e-4, "1"), (2, 60000, 1e-3, "0"),
                                             (4, 200000, 1e-3, "1"), (4, 200000, 1e-3, "0")])
def test_multi_gpu_bit_identical_to_one_gpu(ranks, n, xi, peer):
    """peer = "0": CC_PEER=0 forces the NCCL send/recv + allreduce path of the per-iteration
    exchange instead of the NVLink peer-memory kernel (the fallback is tested)."""
    if torch.cuda.device_count() < ranks:
        pytest.skip(f"needs {ranks} GPUs (tests/test_gpu_vranks.py runs the same protocol on one)")
    env = dict(os.environ, MG_N=str(n), MG_XI=str(xi), CC_PEER=peer)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"ok": true' in r.stdout, r.stdout[-3000:]
