python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import bench_extra as B
for name, env in [("default", {}), ("peel", {"TIDE_SPECULATIVE": "0"}),
                  ("window2", {"TIDE_SPECULATIVE": "0", "TIDE_WINDOW": "2"}),
                  ("window3", {"TIDE_SPECULATIVE": "0", "TIDE_WINDOW": "3"}),
                  ("window2-tailafter1", {"TIDE_SPECULATIVE": "0", "TIDE_WINDOW": "2", "TIDE_TAIL_AFTER": "1"}),
                  ("window4", {"TIDE_SPECULATIVE": "0", "TIDE_WINDOW": "4"})]:
    for k in ("TIDE_SPECULATIVE", "TIDE_WINDOW", "TIDE_TAIL_AFTER"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for th in (0.5, 0.7):
        r = B.config2(th)
        print(name, th, f"graph {r['ms_graph']*1e3:.1f} us exit_rate {r['exit_rate']:.3f}", flush=True)
PY
