#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Produces in gpurun_out/:
#   launches_<tag>.csv   ncu launch list of a short bench run (cold, serialised)
#   prof_<tag>_*.ncu-rep full captures of the top kernels
#   bench_<tag>.json     a real bench line (not under ncu)
TAG=${1:-r01}
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-check > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:route_tc -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_route_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cos_label|decode_tc|route_tcs|select_project|compact_kernel|route_simt|train_act|adam_kernel|route_tf32|chain_resolve" -c 48 \
    -o gpurun_out/prof_${TAG}_aux python tools/profile_aux.py > /dev/null 2>&1
ls -la gpurun_out/
