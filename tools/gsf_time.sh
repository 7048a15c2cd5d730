# time workloads ($WL) through variant libraries of tools/gsf_variants.sh: VARS="a b" WL="c4" bash tools/gsf_time.sh
for w in ${WL:-c4}; do for v in ${VARS}; do
  IGA_LIB_PATH=tune/$v/libiga_b200.so python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-alt 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done; done
