"""N-GPU end-to-end parity of the exchange (NCCL over NVLink). Runs the
worker under torch.distributed.run with one process per visible GPU (2..8);
skipped on a single-GPU box (the single-GPU tests emulate the ranks)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_exchange_multi_gpu():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus N)")
    n = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "mgpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"MGPU world={n}" in r.stdout and "failures=0" in r.stdout


@pytest.mark.gpu
def test_put_one_process_two_gpus():
    """The fused put over real NVLink with loopback windows on two devices of one
    process (scripts/put_nvlink.py): the C2 LLM phase, byte-exact on both ranks."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus N)")
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "scripts",
                                                     "put_nvlink.py"), "2"],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "bytes OK" in r.stdout
