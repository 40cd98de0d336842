"""One launch each of the auxiliary kernels at BASELINE shapes, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_21365_b200 as P
import bench_extra as BE
from oracle import tide_oracle as O
# labeller: 131,072 tokens x d=4096, 8 ckpts + final
n, d = 131072, 4096
fin = torch.randn((n, d), device="cuda").to(torch.bfloat16)
cks = {3 + 4 * i: torch.randn((n, d), device="cuda").to(torch.bfloat16) for i in range(8)}
P.label_tensors(cks, fin, 0.98, labels_dtype="u8")
# decode step (config 3)
ckpts, states, bank = BE._case(36, 4096, 8, torch.bfloat16, 3, 0.3)
P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=0.5))
# peeling chain at the config 2 shape (split-K cluster kernel, 8 links)
ckpts, states, bank = BE._case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=0.5))
# posthoc output staging + compaction + CUDA-core route (config 1, f32)
g = np.random.Generator(np.random.PCG64(42))
routers = {k: O.make_router(768, 128, k, g) for k in (3, 7, 11)}
st = [torch.from_numpy(g.standard_normal((2048, 768), dtype=np.float32)).cuda() for _ in range(13)]
bk = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=12)
head = P.OutputHead(12, 768, np.ones(768, np.float32), np.eye(768, dtype=np.float32)[:256])
P.posthoc_select(head, st, bk, P.RuntimeConfig(exit_threshold=0.5))
m = torch.rand(1 << 20, device="cuda") < 0.4
P.batch_compact(torch.zeros((1 << 20, 8), device="cuda"), m)
torch.cuda.synchronize()
# router training (§8f-4): one epoch at d = 4096 (per-row activation / Adam kernels)
x = torch.randn((4096, 4096), device="cuda")
P.train_router(x, (x[:, 0] > 0).float(), 3, P.CalibrationConfig(epochs=1, batch_size=1024))
# f32 router at 16,384 x 4096: the 64-row CUDA-core kernel, then the opt-in 3xTF32 one
h = torch.randn((16384, 4096), device="cuda")
r = O.make_router(4096, 128, 3, g)
P.route(h, P.Router(layer=3, w_down=r.w_down, w_up=r.w_up), theta=0.5, want_indices=True)
os.environ["TIDE_F32_TC"] = "1"
P.route(h, P.Router(layer=3, w_down=r.w_down, w_up=r.w_up), theta=0.5, want_indices=True)
os.environ.pop("TIDE_F32_TC")
torch.cuda.synchronize()
