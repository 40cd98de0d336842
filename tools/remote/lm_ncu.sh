ncu --set full --clock-control none --import-source on -k regex:lmhead2p_kernel -c 1 -o gpurun_out/prof_r02h_lmhead2p python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B; print(B.lm_head())" > gpurun_out/ncu_lm.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/ncu_lm.log
