timeout 900 python -m pytest tests/test_gpu_posthoc.py tests/test_gpu_route.py tests/test_gpu_advice_r01.py tests/test_hook.py -q -x -p no:cacheprovider --tb=short 2>&1 | tail -4
cat > /tmp/c5.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
import bench_extra as B
for t in (0.5, 0.7):
    r = B.config5(t); print(os.environ.get("TIDE_TCS_GATHER4", "1"), t, f"{r['ms_graph']*1e3:.1f} us", r.get("strategy"), flush=True)
r = B.config2(0.5); print(os.environ.get("TIDE_TCS_GATHER4", "1"), "c2", f"{r['ms_graph']*1e3:.1f} us", flush=True)
PY
for r in 0 1; do for g in 0 1; do TIDE_TCS_GATHER4=$g timeout 300 python /tmp/c5.py 2>&1 | tail -3; done; done
TIDE_SPECULATIVE=0 python -c "
import sys, os; sys.path.insert(0, os.getcwd())
import bench_extra as B
r = B.config2(0.5); print('c2 peel', f\"{r['ms_graph']*1e3:.1f} us\")"
