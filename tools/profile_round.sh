# Capture the round's bench lines, ncu launch lists and full captures (run under gpurun,
# one GPU); summarise with tools/profile_summary.py into profiles/.
TAG=${TAG:-r01k}
set -x
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4.json 2>&1
python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_kron3 --launch-skip 3 -c 1 -f -o gpurun_out/${TAG}_kron python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_k.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_owner.csv python bench.py --assembly owner --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_lo.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gsf3_p3 --launch-skip 3 -c 1 -f -o gpurun_out/${TAG}_owner python bench.py --assembly owner --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_o.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c4.csv python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gsf3_mma --launch-skip 3 -c 1 -f -o gpurun_out/${TAG}_c4 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_c4.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gsf3_mma --launch-skip 3 -c 1 -f -o gpurun_out/${TAG}_c2 python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${TAG}_ncu_c2.log 2>&1
ls -la gpurun_out
