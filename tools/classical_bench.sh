# Algorithm 1 (classical) timings: DMMA kernel vs the scalar kernel (IGA_CLASSICAL_SCALAR=1)
set -x
[ -n "$TESTS" ] && python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in c3 c4 c2; do
  timeout 300 python bench.py --workload $w --method classical --no-alt --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w mma', d['ms_per_step'], d['value'], d['roofline'].get('fp64_frac'))"
  if [ -n "$SCALAR" ]; then IGA_CLASSICAL_SCALAR=1 timeout 300 python bench.py --workload $w --method classical --no-alt --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w scalar', d['ms_per_step'], d['value'])"; fi
done
