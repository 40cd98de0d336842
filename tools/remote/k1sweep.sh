b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], round(d['clocks_sustained']['ms_per_launch']*1e3,1))"; }
for i in 1 2; do
b base
TIDE_NW=3 b nw3
TIDE_NW=2 b nw2
TIDE_K1_NA=3 b na3
done
