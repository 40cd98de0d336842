"""torch.ops.tide.* (the paper's op surface) over the C ABI."""

import numpy as np
import pytest
import torch

from oracle import tide_oracle as O
from tests.gpu_helpers import need_gpu

pytestmark = pytest.mark.gpu


def test_torch_ops_roundtrip():
    need_gpu()
    import paper_2603_21365_b200.torch_ops  # noqa: F401
    g = np.random.Generator(np.random.PCG64(5))
    r = O.make_router(1024, 128, 3, g)
    h = O.round_to(g.standard_normal((3000, 1024), dtype=np.float32), "bf16")
    x = torch.from_numpy(h).cuda().to(torch.bfloat16)
    scores, logits, mask = torch.ops.tide.fused_layernorm_route(
        x, torch.from_numpy(r.w_down).cuda(), torch.from_numpy(r.w_up).cuda(), 1e-6, 0.5)
    _, t_ref, m_ref = O.route_logits(h, r)
    assert O.logits_close(logits.cpu().numpy(), t_ref, m_ref, 2e-2).all()
    ex, co, counts = torch.ops.tide.batch_compact(mask)
    e, c = O.compact_indices(mask.cpu().numpy().astype(bool))
    assert int(counts[0]) == len(e)
    np.testing.assert_array_equal(ex[: len(e)].cpu().numpy(), e)
    np.testing.assert_array_equal(co[: len(c)].cpu().numpy(), c)
    out = torch.zeros((3000, 1024), device="cuda")
    rows = x[torch.from_numpy(e).cuda()]
    torch.ops.tide.exit_scatter(rows, torch.from_numpy(e).cuda(), out)
    assert torch.equal(out[torch.from_numpy(e).cuda()], rows.float())
    gain = torch.ones(1024, device="cuda")
    torch.ops.tide.exit_projection(rows, gain, 1e-6, torch.from_numpy(e).cuda(), out)
    want = np.zeros((3000, 1024), np.float32)
    O.exit_projection(h[e], np.ones(1024, np.float32), 1e-6, e, want)
    np.testing.assert_allclose(out[torch.from_numpy(e).cuda()].cpu().numpy(), want[e],
                               rtol=1e-5, atol=1e-5)
    with pytest.raises(RuntimeError, match="CUDA"):
        torch.ops.tide.batch_compact(mask.cpu())
