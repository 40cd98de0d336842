#!/bin/bash
# Round-2 (second pass) profiling: the bench line after the K1 slot-release
# fix and K1m, the launch list, full ncu captures of K1 (headline) and K1m
# (config 2 speculative, config 5 theta = 1).
TAG=r02b
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-check --no-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_route_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check --no-configs > /dev/null 2>&1
TIDE_CHAIN_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_k1m_c2 python tools/chain_once.py 2 0.5 2 > /dev/null 2>&1
TIDE_CHAIN_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_k1m_c5 python tools/chain_once.py 5 1.0 2 > /dev/null 2>&1
ls -la gpurun_out/ | tail -8
