mkdir -p gpurun_out/ncu_chain
for c in "2 0.5" "2 0.85" "2 1.0" "5 0.7" "5 1.0"; do
  set -- $c
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ncu_chain/c$1_$2.csv python tools/chain_once.py $1 $2 2 > /dev/null 2>&1
done
ls gpurun_out/ncu_chain
