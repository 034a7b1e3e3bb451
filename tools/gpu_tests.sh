# One GPU call: build, then the GPU test suite (optionally a subset: $1 = pytest -k expression).
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$1" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
fi
echo rc=$? >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
