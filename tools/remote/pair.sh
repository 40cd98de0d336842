timeout 600 python -m pytest tests/test_gpu_route.py tests/test_gpu_pdl.py -q -p no:cacheprovider -x 2>&1 | tail -3
for v in 1 0 1 0 1; do
  TIDE_K1_PAIRSLOT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs 2>/dev/null | python -c "
import sys, json; r = json.loads(sys.stdin.read()); print('pair=$v', round(r['ms_per_step']*1e3, 2), 'us', round(r['roofline']['frac'], 4), r['clocks']['sm_mhz'], 'sustained', round(r['clocks_sustained']['ms_per_launch']*1e3,1), r['extra']['kernel_ms_min'])"
done
