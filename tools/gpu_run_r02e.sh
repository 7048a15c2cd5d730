set -x
export IGA_PARITY_LOG=gpurun_out/r02e_parity.jsonl
rm -f $IGA_PARITY_LOG
timeout 1500 python -m pytest tests/test_general_knots_gpu.py -m gpu -q -x --timeout 900 > gpurun_out/r02e_pytest.log 2>&1; tail -40 gpurun_out/r02e_pytest.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02e_pytest_all.log 2>&1; tail -15 gpurun_out/r02e_pytest_all.log
for v in base; do ./build/p3/$v 2>/dev/null; done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02e_bench.json 2>&1; tail -c 600 gpurun_out/r02e_bench.json
