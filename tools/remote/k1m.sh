summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f GB/s %.0f exit %.3f' % (r['ms_graph'], r['ms_api'], r['gbs_graph'], r['exit_rate']), r.get('strategy'), r.get('gbs_read'))"; }
timeout 900 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -x -k "multi or tail_matches or captured or config2 or config5" 2>&1 | tail -5
echo "== default policy"; timeout 600 python bench_extra.py sweep 2>&1 | summ
echo "== peeling"; TIDE_SPECULATIVE=0 timeout 600 python bench_extra.py sweep 2>&1 | summ
