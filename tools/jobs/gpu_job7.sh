ncu --set full --clock-control none -k regex:gather8 -c 1 -o gpurun_out/prof_micro ./tools/l2_gather_bench_v8 > gpurun_out/ncu_micro.log 2>&1
ncu --set full --clock-control none -k regex:k_fwd8 -s 1 -c 1 -o gpurun_out/prof_harness ./tools/fwd_bench > gpurun_out/ncu_harness.log 2>&1
tail -3 gpurun_out/ncu_micro.log gpurun_out/ncu_harness.log
