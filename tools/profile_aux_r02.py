"""One launch each of the kernels added or changed in round 2, at BASELINE
shapes, for ncu: the tensor-core LM head (3-term and hi-only), the wide chain
tail (config 2, theta = 1), the default f32 3xTF32 route (65,536 x 4096), the
u8 exit-code codec + global compaction (8 x 65,536 tokens), the decode step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import numpy as np  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402
from oracle import tide_oracle as O  # noqa: E402
from paper_2603_21365_b200 import _device as Dv, _native as N  # noqa: E402
from paper_2603_21365_b200.runtime import split_bf16  # noqa: E402

lib = N.load()
dev = torch.device("cuda", 0)
s = Dv.stream_handle(dev)
# LM head: 4096 rows x vocab 50,257 x d 4096
n, d, V = 4096, 4096, 50257
a = torch.randn((n, d), device="cuda")
w = torch.randn((V, d), device="cuda") * 0.02
ah, al = split_bf16(a, d)
bh, bl = split_bf16(w, d)
out = torch.empty((n, (V + 3) // 4 * 4), device="cuda")
N.check(lib.tide_lm_head(ah.data_ptr(), al.data_ptr(), d, n, d, bh.data_ptr(), bl.data_ptr(), d,
                         V, out.data_ptr(), out.shape[1], s), "lm3")
N.check(lib.tide_lm_head(ah.data_ptr(), None, d, n, d, bh.data_ptr(), None, d, V,
                         out.data_ptr(), out.shape[1], s), "lm1")
del a, w, ah, al, bh, bl, out
# chain at config 2, theta = 1.0: link 1 + the wide tail + resolve
ckpts, states, bank = BE._case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
os.environ["TIDE_CHAIN_GRAPHS"] = "0"
P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=1.0))
# f32 rows on tcgen05 (3xTF32, 2 accumulators per tile)
g = np.random.Generator(np.random.PCG64(3))
r = O.make_router(4096, 128, 3, g)
h = torch.randn((65536, 4096), device="cuda")
P.route(h, P.Router(layer=3, w_down=r.w_down, w_up=r.w_up), theta=0.5, want_indices=True)
del h
# exit codes of 8 shards + the global compaction (what every rank runs at N = 8)
lay = torch.randint(-1, 80, (8 * 65536,), dtype=torch.int64, device="cuda")
code = torch.empty(8 * 65536, dtype=torch.uint8, device="cuda")
N.check(lib.tide_exit_encode(lay.data_ptr(), lay.numel(), code.data_ptr(), s), "enc")
idx = torch.empty(8 * 65536, dtype=torch.int64, device="cuda")
cnt = torch.empty(2, dtype=torch.int64, device="cuda")
N.check(lib.tide_compact(code.data_ptr(), code.numel(), None, None, 0, None, 0, 0, 0,
                         idx.data_ptr(), None, None, None, cnt.data_ptr(),
                         Dv.workspace(dev).data_ptr(), s), "compact")
# decode step (config 3)
ckpts, states, bank = BE._case(36, 4096, 8, torch.bfloat16, 3, 0.3)
P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=0.5))
torch.cuda.synchronize()
