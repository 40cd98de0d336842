timeout 300 python -m pytest tests/test_gpu_compact_project.py -q -p no:cacheprovider -x 2>&1 | tail -1
ncu --set full --import-source on --clock-control none -k regex:exit_project_staged -c 1 -o gpurun_out/prof_proj2 python tools/project_probe.py > /dev/null 2>&1; ls gpurun_out/prof_proj2.ncu-rep
