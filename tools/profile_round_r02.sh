# Round-2 evidence: bench lines (headline C3 general kernel + separable + e2e + CPU baseline,
# reference arm, C4, C2, p9), ncu launch lists and full captures of the kernels they
# time, GPU suite and smoke.  Run under gpurun (one GPU); summarise with
# tools/profile_summary.py into profiles/.
TAG=${TAG:-r02x}
O=gpurun_out
set -x
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c4.json 2>&1
python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c2.json 2>&1
python bench.py --workload p9 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_p9.json 2>&1
python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c5.json 2>&1
python bench.py --workload c3f --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c3f.json 2>&1
NCUL="ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv"
NCUF="ncu --set full --clock-control none --import-source on --launch-skip 3 -c 1 -f"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$NCUL --log-file $O/${TAG}_launches.csv $B --no-alt > $O/${TAG}_ncu_l.log 2>&1
$NCUF -k regex:k_gsf3_p3 -o $O/${TAG}_p3 $B --no-alt > $O/${TAG}_ncu_p3.log 2>&1
$NCUL --log-file $O/${TAG}_launches_sep.csv $B --assembly separable --no-alt > $O/${TAG}_ncu_ls.log 2>&1
$NCUF -k regex:k_kron3 -o $O/${TAG}_kron $B --assembly separable --no-alt > $O/${TAG}_ncu_k.log 2>&1
$NCUL --log-file $O/${TAG}_launches_c3f.csv $B --workload c3f --no-alt > $O/${TAG}_ncu_l3f.log 2>&1
$NCUF -k regex:k_gsf3_p3 -o $O/${TAG}_c3f $B --workload c3f --no-alt > $O/${TAG}_ncu_c3f.log 2>&1
$NCUL --log-file $O/${TAG}_launches_c4.csv $B --workload c4 --no-alt > $O/${TAG}_ncu_l4.log 2>&1
$NCUF -k regex:k_gsf3_mma -o $O/${TAG}_c4 $B --workload c4 --no-alt > $O/${TAG}_ncu_c4.log 2>&1
$NCUL --log-file $O/${TAG}_launches_c2.csv $B --workload c2 --no-alt > $O/${TAG}_ncu_l2.log 2>&1
$NCUF -k regex:"k_tile3|k_gsf3_mma" -o $O/${TAG}_c2 $B --workload c2 --no-alt > $O/${TAG}_ncu_c2.log 2>&1
export IGA_PARITY_LOG=$O/${TAG}_parity.jsonl
rm -f $IGA_PARITY_LOG
python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; tail -2 $O/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; tail -2 $O/${TAG}_smoke.log
ls -la $O | grep $TAG
