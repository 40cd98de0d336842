summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f' % (r['ms_graph'], r['ms_api']), r.get('strategy'))"; }
timeout 900 python -m pytest tests/test_gpu_posthoc.py tests/test_gpu_route.py -q -p no:cacheprovider -x 2>&1 | tail -2
python tools/timeline_split.py 4096 4096 1 4096 | sed -n "1,14p"
python tools/timeline_split.py 8192 8192 0 | sed -n "9,12p"
cat > /tmp/c5.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
import bench_extra as B
for t in (0.5, 0.7, 0.85):
    print(json.dumps(B.config5(t)))
PY
timeout 300 python /tmp/c5.py 2>&1 | summ
