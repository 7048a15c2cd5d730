# GPU suite + C2 bench through the tile kernel and the streaming kernel (IGA_GSF_TILE=0)
T=${TAG:-t}
if [ -z "$NOTEST" ]; then python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; tail -1 gpurun_out/${T}_pytest.log; fi
for w in ${WL:-c2}; do
  for arm in 1 0; do
    IGA_GSF_TILE=$arm python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${T}_${w}_$arm.json 2>&1
    tail -1 gpurun_out/${T}_${w}_$arm.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w tile=$arm', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
  done
done
