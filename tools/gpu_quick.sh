# quick GPU check: full GPU suite + C2/C4 bench lines (usage: TAG=x bash tools/gpu_quick.sh)
TAG=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for w in c4 c2; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$w.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench_$w.json').readline());print('$w', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c3.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench_c3.json').readline());print('c3', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
