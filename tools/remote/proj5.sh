timeout 300 python -m pytest tests/test_gpu_compact_project.py tests/test_gpu_lmhead.py -q -p no:cacheprovider -x 2>&1 | tail -1
mkdir -p gpurun_out/proj
for st in 0 1; do TIDE_PROJECT_STAGED=$st ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/proj/st$st.csv -k regex:"exit_project" python tools/project_probe.py > /dev/null 2>&1; done
