for v in 1 0 1 0; do TIDE_HOOK_DECODE=$v timeout 600 python tools/hook_bench.py 100 2>&1 | tail -1 | python -c "
import sys, json; r = json.loads(sys.stdin.read()); print('$v', {k: round(v, 1) for k, v in r.items() if k.startswith('us_') or k == 'ms_plain'})"; done
