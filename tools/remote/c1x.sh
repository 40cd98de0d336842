python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import bench_extra as B
for name, env in [("default", {}), ("links-simt", {"TIDE_F32_TAIL_ROWS": "0"}),
                  ("links-tf32", {"TIDE_F32_TAIL_ROWS": "0", "TIDE_F32_TC": "1"}),
                  ("tail-tf32?", {"TIDE_F32_TC": "1"})]:
    for k in ("TIDE_F32_TAIL_ROWS", "TIDE_F32_TC"):
        os.environ.pop(k, None)
    os.environ.update(env)
    r = B.config1()
    print(name, f"api {r['ms_api']*1e3:.1f} us graph {r['ms_graph']*1e3:.1f} us", flush=True)
PY
for tc in 0 1; do TIDE_F32_TC=$tc python tools/tf32_probe.py 2048x768 8192x768 4096x4096 16384x4096 2>&1 | tail -4; done
