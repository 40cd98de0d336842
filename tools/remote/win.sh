summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f GB/s %.0f exit %.3f' % (r['ms_graph'], r['ms_api'], r['gbs_graph'], r['exit_rate']), r.get('strategy'))"; }
timeout 900 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -x 2>&1 | tail -2
for w in 0 2 3 4; do echo "== window $w"; TIDE_WINDOW=$w timeout 600 python bench_extra.py sweep 2>&1 | summ | grep GPU | grep -v "theta=1.0"; done
