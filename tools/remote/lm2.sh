timeout 300 python bench_extra.py lm 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:lmhead -c 2 python bench_extra.py lm 2>&1 | grep -E "lmhead|duration|dram__bytes|tensor" | head -12
