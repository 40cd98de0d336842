TIDE_CHAIN_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:route_tcs_kernel -c 6 \
    -o gpurun_out/prof_r02d_tcs python tools/chain_once.py 5 0.5 1 > /dev/null 2>&1
TIDE_CHAIN_GRAPHS=0 mkdir -p gpurun_out/ncu_chain; ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/ncu_chain/r02d_c5_0.5.csv python tools/chain_once.py 5 0.5 2 > /dev/null 2>&1
ls -la gpurun_out/prof_r02d_tcs.ncu-rep
