timeout 600 python -m pytest tests/test_gpu_route.py tests/test_gpu_posthoc.py -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do for w in 0 1; do TIDE_TCS_WMC=$w timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B
print('wmc=$w', [round(B.config5(t)['ms_graph'], 4) for t in (0.5, 0.7, 0.85)])"; done; done
TIDE_DEBUG_PLAN=1 timeout 120 python tools/timeline_split.py 8192 8192 0 2>&1 | head -12
