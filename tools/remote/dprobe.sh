export TIDE_DEBUG_PLAN=1
python tools/decode_exp.py base 2>&1 | tail -5
for c in 256 512; do TIDE_DECODE_COLS=$c python tools/decode_exp.py cols$c 2>&1 | tail -3; done
for C in 8 9 10 12 16; do python - <<PY 2>&1 | tail -2
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench_extra as BE
import paper_2603_21365_b200 as P
L = 4*$C
ckpts, states, bank = BE._case(L, 4096, 8, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
vals = [BE._graph_time(lambda: P.select_exits(states, bank, cfg), reps=20, inner=20) * 1e3 for _ in range(3)]
print("C", len(ckpts), " ".join(f"{v:.2f}" for v in vals))
PY
done
