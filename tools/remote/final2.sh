timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02d.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['frac_of_8TBs_spec'], d['clocks'], d['clocks_sustained']['ms_per_launch'])
for c in d.get('configs', []): print({k: v for k, v in c.items() if k in ('config', 'ms_graph', 'us_per_step_graph', 'ms', 'ms_3term', 'hbm_frac', 'hbm_frac_read', 'strategy', 'tensor_frac_3term', 'error')})
"
ncu --set full --clock-control none --import-source on -k regex:lmhead2_kernel -c 1 -o gpurun_out/prof_r02d_lmhead2 python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B; B.lm_head()" > /dev/null 2>&1; ls -la gpurun_out/prof_r02d_lmhead2.ncu-rep
