"""Token sharding with the REAL kernels on two ranks.

Two processes share cuda:0 (gloo: NCCL refuses two ranks on one GPU; the
ExitMapGather stages its 1-byte-per-token buffers through the host for
gloo).  Each rank runs the fused route kernel / the select_exits chain on its
contiguous token shard, writing straight into ExitMapGather's send buffer;
after the all-gather every rank derives the global exit indices with one
tide_compact scan.  Checked against

  * the single-process run of the same kernels on each shard (bit-identical
    maps: the kernels are deterministic per row given the shard),
  * the oracle: global decisions within the north_star band, global exit
    indices == the oracle's stable partition of the gathered map (bit-exact).
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import tide_oracle as O

from .gpu_helpers import excused_rows, need_gpu

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _route_case(n, d, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    router = O.make_router(d, 128, 3, g)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
    return router, h


def _chain_case(n, d, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    L = 12
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in ckpts}
    states = [O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
              for _ in range(L + 1)]
    return L, routers, states


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    import paper_2603_21365_b200 as P
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200 import sharding as S

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s0, s1 = S.shard_range(n, rank, world)
        nl = s1 - s0
        # (1) the headline step: fused route kernel -> u8 mask in the send buffer
        router, h = _route_case(n, 4096, 71)
        x = torch.from_numpy(h[s0:s1]).to(dev).to(torch.bfloat16)
        r = P.Router(layer=3, w_down=router.w_down, w_up=router.w_up)
        wd, wu = P.router_ops.device_weights(r, N.BF16, dev)
        gat = S.ExitMapGather(nl, world, dev)
        exit_idx = torch.empty(nl, dtype=torch.int64, device=dev)
        cont_idx = torch.empty(nl, dtype=torch.int64, device=dev)
        counts = torch.empty(2, dtype=torch.int64, device=dev)
        N.check(N.load().tide_route(x.data_ptr(), 4096, nl, None, nl, 4096, N.BF16, None,
                                    wd.data_ptr(), wu.data_ptr(), 128, 1e-6, 0.5, 3, None, None,
                                    gat.exit_map.data_ptr(), exit_idx.data_ptr(),
                                    cont_idx.data_ptr(), 0, None, counts.data_ptr(),
                                    Dv.workspace(dev).data_ptr(), Dv.stream_handle(dev)),
                "tide_route")
        local_mask = gat.exit_map.cpu().numpy().copy()
        local_exit = exit_idx[: int(counts[0])].cpu().numpy()
        gat.all_gather()
        gmask = gat.global_exit_map().cpu().numpy().copy()
        gexit = gat.global_exit_indices().cpu().numpy().copy()
        # (2) config-5 style: the select_exits chain per shard -> u8 exit codes
        L, routers, states = _chain_case(n, 512, 72)
        bank = P.make_bank({k: (rr.w_down, rr.w_up) for k, rr in routers.items()},
                           num_layers=L)
        dstates = [torch.from_numpy(s[s0:s1]).to(dev).to(torch.bfloat16) for s in states]
        gat2 = S.ExitMapGather(nl, world, dev)
        local_layers = S.select_exits_shard(dstates, bank, P.RuntimeConfig(exit_threshold=0.6),
                                            gat2).cpu().numpy()
        glayers = gat2.global_exit_layers().cpu().numpy()
        gexit2 = gat2.global_exit_indices().cpu().numpy().copy()
        torch.cuda.synchronize()
        q.put((rank, local_mask, local_exit, gmask, gexit, local_layers, glayers, gexit2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2 * 3000, 2 * 8192 + 2])
def test_two_ranks_real_kernels_equal_single_process(n):
    need_gpu()
    import torch.multiprocessing as mp

    import paper_2603_21365_b200 as P
    from paper_2603_21365_b200 import sharding as S

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=600)
        res[item[0]] = item[1:]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-process runs of the same kernels on each shard (this process)
    router, h = _route_case(n, 4096, 71)
    L, routers, states = _chain_case(n, 512, 72)
    bank = P.make_bank({k: (rr.w_down, rr.w_up) for k, rr in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=0.6)
    r = P.Router(layer=3, w_down=router.w_down, w_up=router.w_up)
    masks, layers = [], []
    for rank in range(2):
        s0, s1 = S.shard_range(n, rank, 2)
        out = P.route(torch.from_numpy(h[s0:s1]).cuda().to(torch.bfloat16), r, theta=0.5,
                      want_indices=True)
        m = out["mask"].cpu().numpy()
        masks.append(m)
        layers.append(P.select_exits([torch.from_numpy(s[s0:s1]).cuda().to(torch.bfloat16)
                                      for s in states], bank, cfg).cpu().numpy())
        local_mask, local_exit = res[rank][0], res[rank][1]
        assert np.array_equal(local_mask, m)
        assert np.array_equal(local_exit, out["exiting_indices"].cpu().numpy())
        assert np.array_equal(res[rank][4], layers[-1])
    gmask = np.concatenate(masks)
    glayers = np.concatenate(layers)
    # oracle: decisions within the band, stable partition bit-exact
    _, t, mm = O.route_logits(h, router)
    assert O.decision_band_ok(gmask.astype(bool), t, mm, 0.5, 2e-2).all()
    want_exit, _ = O.compact_indices(gmask)
    scores = {k: O.route_logits(states[k + 1], rr)[0] for k, rr in routers.items()}
    want_layers = O.first_exit_from_scores(scores, 0.6)
    exc = excused_rows(states, routers, 0.6, "bf16")
    assert np.array_equal(glayers[~exc], want_layers[~exc])
    for rank in range(2):
        _, _, g_mask, g_exit, _, g_layers, g_exit2 = res[rank]
        assert np.array_equal(g_mask, gmask), f"rank {rank}: gathered mask"
        assert np.array_equal(g_exit, want_exit), f"rank {rank}: global exit indices"
        assert np.array_equal(g_layers, glayers), f"rank {rank}: gathered exit layers"
        assert np.array_equal(g_exit2, np.flatnonzero(glayers >= 0)), f"rank {rank}: C2"


def test_exit_codec_roundtrip():
    need_gpu()
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N

    lib = N.load()
    for n in (0, 1, 1000, 70001):
        lay = torch.randint(-1, 80, (n,), dtype=torch.int64, device="cuda")
        code = torch.empty(n, dtype=torch.uint8, device="cuda")
        back = torch.empty(n, dtype=torch.int64, device="cuda")
        s = Dv.stream_handle(torch.device("cuda", 0))
        N.check(lib.tide_exit_encode(lay.data_ptr(), n, code.data_ptr(), s), "encode")
        N.check(lib.tide_exit_decode(code.data_ptr(), n, back.data_ptr(), s), "decode")
        assert torch.equal(code.cpu().to(torch.int64), lay.cpu() + 1)
        assert torch.equal(back, lay)
