"""Multi-GPU sharded search (a8): bitwise equal to single-GPU (runs only with >= 2 GPUs)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_sharded_topk_bitwise_equals_single_gpu():
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        "--master-port=29533", os.path.join(ROOT, "tests", "dist_topk_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "DIST_OK" in r.stdout
