"""Producer -> route on one stream: the routing kernel must see rows written by
the kernel launched just before it (programmatic dependent launch hazard).

tide_route launches the tensor-core kernel with programmatic stream
serialization, so its CTAs can be resident before the previous kernel on the
stream has finished.  Unless the caller passes TIDE_ROUTE_INPUTS_READY, the
kernel executes griddepcontrol.wait before its first read of h / W_down /
w_up.  Here a torch kernel overwrites h with a different data set right before
every launch (no host sync in between, 200 times); every launch's scores,
mask, exit indices and counts must equal those of a clean, fully synchronised
launch on the same data, which in turn are checked against the oracle
(ee/router_ops.py:68-87 results for the rows just written; SPEC.md:436-437
determinism)."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _device as D
from paper_2603_21365_b200 import _native as N
from oracle import tide_oracle as O
from tests.gpu_helpers import check_decisions, need_gpu

pytestmark = pytest.mark.gpu

N_ROWS, DIM, B, THETA, SETS, ITERS = 16384, 4096, 128, 0.5, 4, 200


@pytest.mark.parametrize("split", ["0", "16"], ids=["persistent", "default-plan"])
@pytest.mark.parametrize("producer", ["copy", "mul"])
def test_rows_written_just_before_route_are_seen(monkeypatch, split, producer):
    need_gpu()
    monkeypatch.setenv("TIDE_SPLIT", split)  # "0": the persistent K1 (route_tc.cu)
    dev = torch.device("cuda", 0)
    g = np.random.Generator(np.random.PCG64(202))
    orouter = O.make_router(DIM, B, 3, g)
    router = P.Router(layer=3, w_down=orouter.w_down, w_up=orouter.w_up)
    wd, wu = P.router_ops.device_weights(router, N.BF16, dev)
    gen = torch.Generator(device=dev)
    sets = []
    for s in range(SETS):
        gen.manual_seed(77 + s)
        # alternate scales so a stale read of the previous set changes decisions
        sets.append((torch.randn((N_ROWS, DIM), generator=gen, device=dev) *
                     (1.0 + s)).to(torch.bfloat16))
    h = torch.empty((N_ROWS, DIM), dtype=torch.bfloat16, device=dev)
    lib = N.load()
    st = torch.cuda.current_stream(dev)
    sh = st.cuda_stream
    ws = D.workspace(dev).data_ptr()

    def produce(j):
        if producer == "copy":
            h.copy_(sets[j])
        else:
            torch.mul(sets[j], 1.0, out=h)

    def launch(scores, mask, eidx, cidx, cnt):
        rc = lib.tide_route(h.data_ptr(), DIM, N_ROWS, None, N_ROWS, DIM, N.BF16, None,
                            wd.data_ptr(), wu.data_ptr(), B, 1e-6, THETA, 3, scores.data_ptr(),
                            None, mask.data_ptr(), eidx.data_ptr(), cidx.data_ptr(), 0, None,
                            cnt.data_ptr(), ws, sh)
        if rc:
            N.check(rc, "tide_route")

    def bufs(k):
        return (torch.empty((k, N_ROWS), dtype=torch.float32, device=dev),
                torch.empty((k, N_ROWS), dtype=torch.uint8, device=dev),
                torch.empty((k, N_ROWS), dtype=torch.int64, device=dev),
                torch.empty((k, N_ROWS), dtype=torch.int64, device=dev),
                torch.empty((k, 2), dtype=torch.int64, device=dev))

    # clean results: producer, full sync, route, full sync
    clean = bufs(SETS)
    for j in range(SETS):
        produce(j)
        torch.cuda.synchronize(dev)
        launch(*(b[j] for b in clean))
        torch.cuda.synchronize(dev)
        # the clean launch itself against the oracle (first 1,024 rows: band
        # rule on decisions; compaction bit-exact on the GPU's own mask)
        hs = sets[j][:1024].float().cpu().numpy()
        _, t_ref, m_ref = O.route_logits(hs, orouter)
        check_decisions(clean[1][j][:1024].cpu().numpy(), t_ref, m_ref, THETA, "bf16",
                        f"set {j}")
        e, c = O.compact_indices(clean[1][j].cpu().numpy())
        ne = int(clean[4][j][0])
        np.testing.assert_array_equal(clean[2][j][:ne].cpu().numpy(), e)
        np.testing.assert_array_equal(clean[3][j][:N_ROWS - ne].cpu().numpy(), c)
    # the data sets must really differ in their decisions
    assert len({int(clean[4][j][0]) for j in range(SETS)}) > 1

    out = bufs(ITERS)
    torch.cuda.synchronize(dev)
    for i in range(ITERS):
        produce(i % SETS)  # a torch kernel writes h ...
        launch(*(b[i] for b in out))  # ... and the route is queued right behind it
    torch.cuda.synchronize(dev)
    idx = torch.arange(ITERS, device=dev) % SETS
    bad = []
    for name, got, want in zip(("scores", "mask", "exit_idx", "cont_idx", "counts"), out, clean):
        ref = want[idx]
        if name in ("exit_idx", "cont_idx"):
            # only the first counts entries are defined
            ne = clean[4][:, 0][idx]
            k = ne if name == "exit_idx" else N_ROWS - ne
            col = torch.arange(N_ROWS, device=dev)[None, :]
            valid = col < k[:, None]
            diff = ((got != ref) & valid).any(dim=1)
        else:
            diff = (got != ref).reshape(ITERS, -1).any(dim=1)
        if bool(diff.any()):
            bad.append((name, diff.nonzero().flatten()[:10].tolist()))
    assert not bad, f"launches that read stale rows: {bad}"
