# time C4/C2 through each variant library in tune/ (usage: bash tools/gpu_var.sh "c4 c2" v1 v2 ...)
W=$1; shift
for v in "$@"; do for w in $W; do
  IGA_LIB_PATH=tune/$v/libiga_b200.so python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/var_${v}_$w.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/var_${v}_$w.json').readline());print('$v $w', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))" || tail -3 gpurun_out/var_${v}_$w.json
done; done
