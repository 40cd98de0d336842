"""Which (group ordinal in the CTA, tile in group) K1 outputs differ between
repeated launches (debug of the multi-group race): python tools/stress_detail.py n d reps"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_21365_b200 as P
n, d = int(sys.argv[1]), int(sys.argv[2])
g = np.random.Generator(np.random.PCG64(n + d))
wd = (g.standard_normal((128, d)) * 0.05).astype(np.float32)
wu = (g.standard_normal((1, 128)) * 0.05).astype(np.float32)
router = P.Router(layer=3, w_down=wd, w_up=wu)
h = torch.randn((n, d), device="cuda").to(torch.bfloat16)
# exact reference logits (f64 on device)
ref = P.route(h, router, theta=0.5, want_logits=True)["logits"].clone()
tiles = (n + 127) // 128; NG = max(min(tiles, 148), (tiles + 3) // 4)
G = 148
def grp(tile):
    for gg in range(NG):
        r0 = gg * tiles // NG; r1 = (gg + 1) * tiles // NG
        if r0 <= tile < r1: return gg, tile - r0, r1 - r0
from collections import Counter
cnt = Counter()
junk = torch.empty(1 << 26, device="cuda")
for rep in range(int(sys.argv[3])):
    junk.fill_(float(rep))
    r = P.route(h, router, theta=0.5, want_logits=True)
    bad = torch.nonzero(r["logits"] != ref).flatten().cpu().numpy()
    for t in sorted(set((bad // 128).tolist())):
        gg, tt, T = grp(t)
        rows = int(((bad // 128) == t).sum())
        cnt[(gg // G, tt, T, rows == 128)] += 1
print("(group ordinal in CTA, tile in group, T, whole tile) -> count:")
for k, v in sorted(cnt.items()): print(k, v)
