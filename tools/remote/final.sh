timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python tools/stress_k1.py 60 160000x2048 94720x128 65536x4096 2>&1 | grep reps
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02c.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['frac_of_8TBs_spec'], d['clocks'], d['clocks_sustained']['ms_per_launch'])
for c in d.get('configs', []): print({k: v for k, v in c.items() if k in ('config', 'ms_graph', 'us_per_step_graph', 'ms', 'hbm_frac', 'hbm_frac_read', 'strategy', 'tensor_frac_3term', 'error')})
"
