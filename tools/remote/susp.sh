b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], round(d['clocks_sustained']['ms_per_launch']*1e3,1))"; }
cp paper_2603_21365_b200/_lib/libtide_b200.so /tmp/base.so
for i in 1 2; do
  cp /tmp/base.so paper_2603_21365_b200/_lib/libtide_b200.so; b base1000
  for v in 0 250 500 2000; do cp tools/_libs/susp$v.so paper_2603_21365_b200/_lib/libtide_b200.so; b susp$v; done
done
cp /tmp/base.so paper_2603_21365_b200/_lib/libtide_b200.so
