python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import bench_extra as B
for name, env in [("wide (64-row)", {}), ("16-row", {"TIDE_F32_TAIL_WIDE": "0"})]:
    os.environ.pop("TIDE_F32_TAIL_WIDE", None)
    os.environ.update(env)
    for _ in range(2):
        r = B.config1()
        print(name, f"api {r['ms_api']*1e3:.1f} us graph {r['ms_graph']*1e3:.1f} us", flush=True)
PY
