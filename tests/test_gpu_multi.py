"""Multi-GPU runner (NCCL round boundary): results must not depend on the GPU
count.  Launched by this test as `torchrun --nproc-per-node 2` when >= 2 GPUs
are visible (gpurun --gpus 2); each rank's theta after R rounds must equal the
single-GPU runner's theta bit for bit (same kernels, same ascending-order
aggregation arithmetic, f32 mode), and so must the per-round evaluation (eval
batches sharded over ranks) and the saved resume directory."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = os.path.join(ROOT, "tools", "multi_rank_check.py")


CASES = [(s, "auto") for s in ("fedavg", "diloco", "diloco_drop", "central", "diloco_many")] + \
        [(s, b) for s in ("fedavg", "diloco", "diloco_k8") for b in ("p2p", "nccl")]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("server,boundary", CASES)
def test_world_size_invariance(tmp_path, server, boundary):
    """Both boundary paths (NVLink peer-memory kernel, NCCL send/recv + fused
    update + all-gather; PHOTON_BOUNDARY forces one) and 1 / 2 local clients
    per rank give theta bit-identical to one GPU."""
    n = min(torch.cuda.device_count(), 4)
    out1 = tmp_path / "w1.npy"
    outn = tmp_path / "wn.npy"
    env = dict(os.environ, PYTHONPATH=ROOT)
    if boundary != "auto":
        env["PHOTON_BOUNDARY"] = boundary
    r = subprocess.run([sys.executable, SCRIPT, str(out1), server], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", SCRIPT, str(outn), server],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    a, b = np.load(out1), np.load(outn)
    assert a.tobytes() == b.tobytes()  # theta, velocity and the per-round eval ppls
    assert np.all(np.isfinite(a))
    if server == "central":
        return
    for f in ("checkpoint.phck", "state.json") + (("velocity.phck",) if "diloco" in server else ()):
        assert open(str(out1) + ".ckpt/" + f, "rb").read() == open(str(outn) + ".ckpt/" + f,
                                                                     "rb").read()
