summ() { python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'][-32:], 'ms_graph %.4f api %.4f' % (r['ms_graph'], r['ms_api']), r.get('strategy'))"; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_floor tools/pdl_floor.cu && ./tools/pdl_floor
cat > /tmp/c5.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
import bench_extra as B
for t in (0.5, 0.7):
    print(json.dumps(B.config5(t)))
PY
for a in 2 3 4 5; do for ks in 2 4; do echo "== TAIL_AFTER=$a TAIL_KS=$ks"; TIDE_TAIL_AFTER=$a TIDE_TAIL_KS=$ks timeout 300 python /tmp/c5.py 2>&1 | summ; done; done
for rows in 1024 4096; do echo "== TAIL_ROWS=$rows"; TIDE_TAIL_ROWS=$rows timeout 300 python /tmp/c5.py 2>&1 | summ; done
