set -x
export IGA_PARITY_LOG=gpurun_out/r02c_parity.jsonl
rm -f $IGA_PARITY_LOG
timeout 1500 python -m pytest tests/test_high_degree_gpu.py tests/test_dropin_gpu.py -m gpu -q --timeout 900 > gpurun_out/r02c_pytest.log 2>&1; tail -30 gpurun_out/r02c_pytest.log
timeout 600 python bench.py --workload p9 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_p9.json 2> gpurun_out/r02c_bench_p9.err; tail -c 2500 gpurun_out/r02c_bench_p9.json; tail -5 gpurun_out/r02c_bench_p9.err
timeout 600 python bench.py --workload p9 --method classical --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02c_bench_p9_classical.json 2>&1; tail -c 1500 gpurun_out/r02c_bench_p9_classical.json
