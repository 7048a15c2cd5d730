set -x
export IGA_PARITY_LOG=gpurun_out/r02b_parity.jsonl
rm -f $IGA_PARITY_LOG
timeout 1500 python -m pytest tests/test_multirank_gpu.py tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "multirank or reproducible or slab or devices or full_size_c3 or sampled_rows" > gpurun_out/r02b_pytest.log 2>&1; tail -30 gpurun_out/r02b_pytest.log
