#!/bin/bash
# Round-2 profiling pass (run under gpurun, 1 GPU): a real bench line (not
# under ncu), the launch list of a short bench run, full ncu captures of K1
# and of the round-2 kernels.
TAG=r02
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-check --no-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_route_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check --no-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"lmhead|route_tcs|chain_resolve|route_tf32|exit_encode|compact_kernel|decode_tc" -c 12 \
    -o gpurun_out/prof_${TAG}_aux python tools/profile_aux_r02.py > gpurun_out/prof_${TAG}_aux.log 2>&1
ls -la gpurun_out/ | tail -12
