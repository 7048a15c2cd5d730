# source-level ncu captures of k_gsf3_p3 harness builds (tools/p3_time.cu): V="bonly full"
for v in $V; do
  ncu --set full --clock-control none --import-source on -k regex:k_gsf3_p3 --launch-skip 2 -c 1 -f -o gpurun_out/p3_$v ./build/p3/$v > gpurun_out/p3_$v.log 2>&1
done
ls -la gpurun_out | grep p3_
