timeout 300 python -m pytest tests/test_gpu_compact_project.py -q -p no:cacheprovider -x -k "staged and f32-8" 2>&1 | grep -E "^E" | head -12
mkdir -p gpurun_out/proj
for st in 0 1; do TIDE_PROJECT_STAGED=$st ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/proj/st$st.csv -k regex:"exit_project|select_project" python tools/project_probe.py > /dev/null 2>&1; done
ls gpurun_out/proj
