summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f GB/s %.0f exit %.3f' % (r['ms_graph'], r['ms_api'], r['gbs_graph'], r['exit_rate']), r.get('strategy'))"; }
timeout 900 python -m pytest tests/test_gpu_posthoc.py tests/test_gpu_route.py -q -p no:cacheprovider -x 2>&1 | tail -2
python tools/timeline_split.py 4096 4096 1 4096 2>/dev/null | head -12
python tools/timeline_split.py 8192 8192 0 2>/dev/null | head -8
echo "== sweep"; timeout 600 python bench_extra.py sweep 2>&1 | summ | grep GPU
