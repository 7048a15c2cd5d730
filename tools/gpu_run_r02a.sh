set -x
export IGA_PARITY_LOG=gpurun_out/r02a_parity.jsonl
rm -f $IGA_PARITY_LOG
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02a_pytest.log 2>&1; tail -15 gpurun_out/r02a_pytest.log
