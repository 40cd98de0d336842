for L in 24 28 32 36 40; do python -c "
import os, sys; sys.path.insert(0, '.')
import torch, bench_extra as BE, paper_2603_21365_b200 as P
ckpts, states, bank = BE._case($L, 4096, 8, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
v = [BE._graph_time(lambda: P.select_exits(states, bank, cfg), reps=20, inner=20) * 1e3 for _ in range(3)]
print('C =', len(ckpts), ' '.join(f'{x:.2f}' for x in v), 'us/step')"; done
