set -x
python __graft_entry__.py > gpurun_out/r02b_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02b_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02b_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_c3.json 2> gpurun_out/r02b_c3.err
timeout 600 python bench.py --workload config5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_c5.json 2> gpurun_out/r02b_c5.err
