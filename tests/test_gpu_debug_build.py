"""The device-assert build (libhiper_debug.so, -DHIPER_DEVICE_ASSERTS) -- the stand-in for
compute-sanitizer, which this pool does not offer.  It re-runs a cross-section of the GPU parity
suite (dense, packed and pooled top-k, the key merge, two-stage retrieval at k1 = 100, the N2 gather)
with every device-side bound check compiled in: any out-of-range index traps and fails the run."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_parity_subset_under_device_asserts():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2505_04846_b200", "libhiper_debug.so")
    if not os.path.exists(lib):
        pytest.skip("libhiper_debug.so not built (__graft_entry__.build())")
    env = dict(os.environ, HIPER_LIB="debug")
    sel = ["tests/test_gpu_shard_merge.py", "tests/test_gpu_rerank.py", "tests/test_gpu_packed.py",
           "tests/test_gpu_parity.py::test_topk_config1", "tests/test_gpu_pooled.py::test_pooled_topk",
           "tests/test_gpu_coltrast_full.py::test_full_coltrast_loss_simulated_ranks"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        *sel], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, "debug-build run failed"
    which = subprocess.run([sys.executable, "-c", "import paper_2505_04846_b200 as H; H.lib(); print(H.LIB_PATH)"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=300).stdout
    assert which.strip().endswith("libhiper_debug.so"), which
