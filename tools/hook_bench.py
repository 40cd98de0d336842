"""§8f-2 measurement: checkpoint capture + exit decision on a torch decoder at
batch-8 decode (the setting where the paper reports that collecting every
hidden state is the bottleneck).

Model: a Llama-8B-shaped decoder in plain PyTorch (d=4096, 32 layers, 32
heads / 8 KV heads, SwiGLU MLP 14336, RMSNorm; random init, bf16) with a
static 512-token KV cache, so that one decode step (batch 8, one token per
sequence) can be captured in a CUDA graph: the numbers are GPU time per step
(CUDA events over graph replays), free of Python/launch overhead.  Bank: 8
checkpoint routers (every 4th layer, b=128).  Variants, each one graph:

  plain     the decoder step alone (no exit logic)
  full      every layer's output copied out (output_hidden_states) + select_exits
            over all L+1 states (the reference's flow: capture everything, then route)
  capture   CheckpointCapture hooks (checkpoint layers only, no copies) + select_exits
  online    CheckpointCapture(online=True): routing inside the hooks (decode-sized
            batch: one decode-kernel launch in the last checkpoint's hook;
            TIDE_HOOK_DECODE=0: one link launch per checkpoint)

    python tools/hook_bench.py [replays]
"""

import json
import os
import sys

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402
from paper_2603_21365_b200.hook import CheckpointCapture  # noqa: E402
from oracle import tide_oracle as O  # noqa: E402

D, L, H, KVH, FF, CTX, B = 4096, 32, 32, 8, 14336, 512, 8
HD = D // H


class Layer(nn.Module):
    def __init__(self):
        super().__init__()
        s = D ** -0.5
        self.qkv = nn.Parameter(torch.randn(D + 2 * KVH * HD, D) * s)
        self.o = nn.Parameter(torch.randn(D, D) * s)
        self.gu = nn.Parameter(torch.randn(2 * FF, D) * s)
        self.down = nn.Parameter(torch.randn(D, FF) * FF ** -0.5)
        self.n1 = nn.Parameter(torch.ones(D))
        self.n2 = nn.Parameter(torch.ones(D))
        self.k = torch.randn(B, KVH, CTX, HD)  # static KV cache (random past)
        self.v = torch.randn(B, KVH, CTX, HD)

    def forward(self, x):  # x [B, 1, D]
        h = F.rms_norm(x, (D,), self.n1)
        q, k, v = (h @ self.qkv.t()).split([D, KVH * HD, KVH * HD], dim=-1)
        q = q.view(B, 1, H, HD).transpose(1, 2)
        k = torch.cat([self.k, k.view(B, 1, KVH, HD).transpose(1, 2)], dim=2)
        v = torch.cat([self.v, v.view(B, 1, KVH, HD).transpose(1, 2)], dim=2)
        a = F.scaled_dot_product_attention(q, k, v, enable_gqa=True)
        x = x + a.transpose(1, 2).reshape(B, 1, D) @ self.o.t()
        g, u = (F.rms_norm(x, (D,), self.n2) @ self.gu.t()).chunk(2, dim=-1)
        return (x + (F.silu(g) * u) @ self.down.t(),)  # HF-style tuple


class Decoder(nn.Module):
    def __init__(self):
        super().__init__()
        self.model = nn.Module()
        self.model.layers = nn.ModuleList([Layer() for _ in range(L)])
        self.keep = None  # static buffer for the "full" capture variant

    def forward(self, x, keep_all=False):
        if keep_all:
            self.keep[0].copy_(x.view(B, D))
        for i, layer in enumerate(self.model.layers):
            x = layer(x)[0]
            if keep_all:
                self.keep[i + 1].copy_(x.view(B, D))
        return x


def make_graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
    return g, s, out


def time_graph(g, s, replays):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(replays):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / replays


def main(replays=50):
    torch.manual_seed(0)
    torch.set_default_dtype(torch.bfloat16)
    with torch.device("cuda"):
        model = Decoder().eval()
        model.keep = torch.empty(L + 1, B, D)
        x = torch.randn(B, 1, D)
    torch.set_default_dtype(torch.float32)
    g = np.random.Generator(np.random.PCG64(7))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(D, 128, k, g, scale=0.05) for k in ckpts}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=0.6)
    graphs, maps = {}, {}
    with torch.no_grad():
        graphs["plain"] = make_graph(lambda: model(x))

        def full():
            model(x, keep_all=True)
            return P.select_exits(list(model.keep), bank, cfg)
        graphs["full"] = make_graph(full)

        cap = CheckpointCapture(model, bank.checkpoints)

        def capture():
            with cap:
                model(x)
            return P.select_exits(cap.hidden_states, bank, cfg)
        graphs["capture"] = make_graph(capture)

        ocap = CheckpointCapture(model, bank.checkpoints, bank=bank, config=cfg, online=True)

        def online():
            with ocap:
                model(x)
            return ocap.exit_layers
        graphs["online"] = make_graph(online)
    for k, (_, _, out) in graphs.items():
        if k != "plain":
            maps[k] = out
    # interleaved rounds, median per variant (single runs vary by tens of us)
    rounds = {k: [] for k in graphs}
    for _ in range(7):
        for k, (g, st, _) in graphs.items():
            rounds[k].append(time_graph(g, st, replays))
    res = {k: float(np.median(v)) for k, v in rounds.items()}
    res["plain_again"] = res["plain"]
    base = min(res["plain"], res["plain_again"])
    m = {k: v.cpu().numpy() for k, v in maps.items()}
    weights = sum(p.numel() * p.element_size() for p in model.parameters())
    print(json.dumps({
        "what": "batch-8 decode step, Llama-8B-shaped decoder (d=4096, 32 layers, GQA 32/8, "
                "MLP 14336, bf16, random init, static 512-token KV cache), 8 checkpoint routers; "
                "GPU ms per step (CUDA-graph replays)",
        "ms_plain": base, "ms_full_capture_plus_select": res["full"],
        "ms_checkpoint_capture_plus_select": res["capture"], "ms_online_routing": res["online"],
        "us_overhead_full": 1e3 * (res["full"] - base),
        "us_overhead_capture": 1e3 * (res["capture"] - base),
        "us_overhead_online": 1e3 * (res["online"] - base),
        "rounds_ms": {k: [round(x, 4) for x in v] for k, v in rounds.items()},
        "weights_gb": weights / 1e9, "plain_gbs": weights / (base / 1e3) / 1e9,
        "exit_maps_equal": bool(np.array_equal(m["full"], m["capture"])
                                and np.array_equal(m["full"], m["online"])),
        "exit_rate": float((m["full"] >= 0).mean())}), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 50)
