"""Multi-process (world_size 2, gloo, CPU) test of the token-sharding host
logic: contiguous shards, C1 exit-map all-gather, C2 compacted-index
assembly.  The per-rank compute is the oracle here (no GPU); on B200 the
same host code wraps the kernels with NCCL (tests/test_gpu_sharding.py runs
the real kernels through it on two ranks).  The gathered result must be
bit-identical to the single-process partition."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_21365_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compactor(mask, out_idx, counts):
    """The CPU tests' stand-in for tide_compact (the oracle's stable partition)."""
    from oracle import tide_oracle as O
    e, c = O.compact_indices(mask.numpy())
    out_idx[: len(e)] = torch.from_numpy(e)
    counts.copy_(torch.tensor([len(e), len(c)], dtype=torch.int64))


def _worker(rank, world, port, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.random.Generator(np.random.PCG64(seed))
        mask_all = g.random(n) < 0.4
        layer_all = np.where(mask_all, 7, -1).astype(np.int64)
        s0, s1 = S.shard_range(n, rank, world)
        local_mask = mask_all[s0:s1]
        # per-rank stable partition (what tide_route writes per shard)
        idx = np.arange(s1 - s0, dtype=np.int64)
        e, c = idx[local_mask], idx[~local_mask]
        n_local = s1 - s0
        if n % world == 0:
            gat = S.ExitMapGather(n_local, world, "cpu", compactor=_oracle_compactor)
            # what tide_route writes into the send buffer: the shard's u8 mask
            gat.exit_map.copy_(torch.from_numpy(local_mask.astype(np.uint8)))
            gat.all_gather()
            glob_exit = gat.global_exit_indices().numpy().copy()
            glob_map = gat.global_exit_map().numpy().astype(bool)
            # exit codes of a multi-checkpoint map: encode -> gather -> decode
            gat.encode(torch.from_numpy(layer_all[s0:s1]))
            gat.all_gather()
            glob_codes = gat.global_exit_layers().numpy()
            glob_code_exit = gat.global_exit_indices().numpy().copy()
            assert np.array_equal(glob_codes, layer_all)
            assert np.array_equal(glob_code_exit, glob_exit)
        else:
            glob_exit = None
            glob_map = None
        glob_layers = S.gather_exit_layers(torch.from_numpy(layer_all[s0:s1]), world).numpy()
        # host C2 assembly from all ranks' lists
        lists = [None] * world
        dist.all_gather_object(lists, (e, c, s0))
        ge, gc = S.assemble_partition(
            [(torch.from_numpy(a), torch.from_numpy(b)) for a, b, _ in lists],
            [(len(a), len(b)) for a, b, _ in lists], [o for _, _, o in lists])
        if rank == 0:
            q.put((glob_exit, glob_map, glob_layers, ge.numpy(), gc.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 1001, 65536])
def test_two_rank_gather_equals_single_process(n):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    seed = 11 + n
    ctxs = mp.start_processes(_worker, args=(2, port, n, seed, q), nprocs=2, join=False,
                              start_method="spawn")
    glob_exit, glob_map, glob_layers, ge, gc = q.get()  # read before join: pipe would block
    while not ctxs.join(timeout=60):
        pass
    g = np.random.Generator(np.random.PCG64(seed))
    mask = g.random(n) < 0.4
    idx = np.arange(n, dtype=np.int64)
    np.testing.assert_array_equal(ge, idx[mask])
    np.testing.assert_array_equal(gc, idx[~mask])
    np.testing.assert_array_equal(glob_layers, np.where(mask, 7, -1))
    if glob_exit is not None:
        np.testing.assert_array_equal(glob_exit, idx[mask])
        np.testing.assert_array_equal(glob_map, mask)


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            rs = [S.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _label_worker(rank, world, port, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tide_oracle as O
        g = np.random.Generator(np.random.PCG64(seed))
        d = 32
        fin = g.standard_normal((n, d), dtype=np.float32)
        cks = {k: (fin + g.standard_normal((n, d), dtype=np.float32) * s).astype(np.float32)
               for k, s in ((3, 0.1), (7, 0.5), (11, 2.0))}
        cks[7][::50] = 0.0  # zero-norm rows
        s0, s1 = S.shard_range(n, rank, world)

        def oracle_labeller(ck, f, tau):
            lab, sims, _ = O.compute_labels(ck, f, tau)
            ks = tuple(ck)
            zero = torch.tensor([int(((np.linalg.norm(ck[k], axis=1) == 0)
                                      | (np.linalg.norm(f, axis=1) == 0)).sum()) for k in ks])
            return (ks, torch.from_numpy(np.stack([sims[k] for k in ks])),
                    torch.from_numpy(np.stack([lab[k] for k in ks]).astype(np.uint8)), zero)

        out = S.label_shard({k: v[s0:s1] for k, v in cks.items()}, fin[s0:s1], 0.9, world,
                            gather=True, labeller=oracle_labeller)
        if rank == 0:
            lab, _, zt = O.compute_labels(cks, fin, 0.9)
            want = np.stack([lab[k] for k in (3, 7, 11)]).astype(np.uint8)
            q.put((out["global_labels"].numpy(), want, out["zero_counts"].numpy(),
                   out["positives"].numpy(), zt))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [999, 1000])
def test_two_rank_labelling_equals_single_process(n):
    """Config 4 sharded: gathered labels == the single-process labels; the
    all-reduced zero-norm and positive counts == the global ones."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_label_worker, args=(r, 2, port, n, 31, q)) for r in range(2)]
    for p in ps:
        p.start()
    got, want, zero, pos, zt = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(got, want)
    assert int(zero.sum()) == zt
    np.testing.assert_array_equal(pos, want.sum(axis=1))
