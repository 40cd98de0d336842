python tools/tf32_probe.py 65536x4096 > gpurun_out/tf32_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:route_tf32_kernel -s 3 -c 1 -o gpurun_out/prof_r02j_tf32 python tools/tf32_probe.py 65536x4096 > gpurun_out/ncu_tf32.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_tf32.log
