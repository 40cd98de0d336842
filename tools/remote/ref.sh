timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import sys, json; r = json.loads(sys.stdin.read()); print(json.dumps({k: r[k] for k in ('value', 'ms_per_step', 'cpu_baseline', 'e2e', 'roofline')}))"
