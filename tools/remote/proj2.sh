timeout 300 python -m pytest tests/test_gpu_compact_project.py tests/test_gpu_lmhead.py -q -p no:cacheprovider -x 2>&1 | tail -2
TIDE_PROJECT_STAGED=1 ncu --set full --import-source on --clock-control none -k regex:exit_project -c 1 -o gpurun_out/prof_proj python tools/project_probe.py > /dev/null 2>&1; ls -la gpurun_out/prof_proj.ncu-rep
