timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/r02j_pytest.log 2>&1; tail -3 gpurun_out/r02j_pytest.log
ncu --set full --clock-control none --import-source on -k regex:k_gsf3_mma --launch-skip 3 -c 1 -f -o gpurun_out/r02j_c4 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02j_ncu_c4.log 2>&1
tail -2 gpurun_out/r02j_ncu_c4.log
