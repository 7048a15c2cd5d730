# full ncu captures (with source) of the generic DMMA kernel on C4 and C2
O=gpurun_out
NCUF="ncu --set full --clock-control none --import-source on --launch-skip 3 -c 1 -f"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-alt"
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > $O/${TAG}_bench_c4.json 2>&1
python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > $O/${TAG}_bench_c2.json 2>&1
$NCUF -k regex:k_gsf3_mma -o $O/${TAG}_c4 $B --workload c4 > $O/${TAG}_ncu_c4.log 2>&1
$NCUF -k regex:k_gsf3_mma -o $O/${TAG}_c2 $B --workload c2 > $O/${TAG}_ncu_c2.log 2>&1
ls -la $O | grep $TAG
