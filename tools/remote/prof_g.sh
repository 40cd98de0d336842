# round-2g profiles at HEAD: launch list of the bench command, one --set full capture of K1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02g.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs \
  > gpurun_out/ncu_list_r02g.log 2>&1; echo "list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 5 -c 1 -o gpurun_out/prof_r02g_k1 \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ncu_full_r02g.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/
