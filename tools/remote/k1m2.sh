summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f GB/s %.0f exit %.3f' % (r['ms_graph'], r['ms_api'], r['gbs_graph'], r['exit_rate']), r.get('strategy'), r.get('gbs_read'))"; }
timeout 900 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -x 2>&1 | tail -2
echo "== default policy"; timeout 600 python bench_extra.py sweep 2>&1 | summ
mkdir -p gpurun_out/ncu_chain
for c in "2 0.5" "5 0.5" "5 1.0"; do set -- $c; ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ncu_chain/k1m_c$1_$2.csv python tools/chain_once.py $1 $2 2 > /dev/null 2>&1; done
