"""Token sharding across the GPUs of one box.

Every per-token quantity on this path is row-independent, so rank r owns the
contiguous token range shard_range(n, r, R) and runs the kernels on it with no
exchange during compute.  The only collectives are

  C1  all-gather of the per-token exit map (u8 mask or int64 exit layer), and
  C2  all-gather of the per-rank stable partitions (counts + padded index
      lists); because shards are contiguous and in rank order, the GLOBAL
      stable partition is the concatenation of the per-rank ones with the
      rank offsets added — bit-identical to the single-GPU result by
      construction.

Backend-agnostic (NCCL on GPUs, gloo on CPU for the host-logic tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous [start, end) of rank `rank`; sizes differ by at most one."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class ExitMapGather:
    """C1 + C2 as ONE all-gather per step for equal shards of n_local tokens.

    Each rank's send buffer packs [counts int64 x2 | exit indices int64 x
    n_local | exit map u8 x n_local]; the route kernel writes its outputs
    straight into those views (`counts`, `exit_idx`, `exit_map`), so the
    exchange is a single collective with no packing copies."""

    def __init__(self, n_local: int, world: int, device, group=None):
        self.n_local = n_local
        self.world = world
        self.group = group
        self.nbytes = 16 + 8 * n_local + ((n_local + 15) // 16) * 16
        self.send = torch.zeros(self.nbytes, dtype=torch.uint8, device=device)
        self.recv = torch.empty(world * self.nbytes, dtype=torch.uint8, device=device)
        self.counts = self.send[:16].view(torch.int64)
        self.exit_idx = self.send[16:16 + 8 * n_local].view(torch.int64)
        self.exit_map = self.send[16 + 8 * n_local:16 + 9 * n_local]

    def all_gather(self, async_op: bool = False):
        return dist.all_gather_into_tensor(self.recv, self.send, group=self.group,
                                           async_op=async_op)

    def _rank_views(self, r):
        base = r * self.nbytes
        blk = self.recv[base:base + self.nbytes]
        return (blk[:16].view(torch.int64), blk[16:16 + 8 * self.n_local].view(torch.int64),
                blk[16 + 8 * self.n_local:16 + 9 * self.n_local])

    def global_exit_map(self) -> torch.Tensor:
        """C1: the exit map of all ranks' shards, in token order."""
        return torch.cat([self._rank_views(r)[2] for r in range(self.world)])

    def global_exit_indices(self) -> torch.Tensor:
        """C2: concatenate the per-rank stable exit lists with rank offsets."""
        parts = []
        for r in range(self.world):
            cnt, idx, _ = self._rank_views(r)
            k = int(cnt[0])
            parts.append(idx[:k] + r * self.n_local)
        return torch.cat(parts) if parts else self.exit_idx[:0]


def assemble_partition(local_lists, local_counts, offsets):
    """Host-side C2 assembly from per-rank (exit_idx, cont_idx) lists.

    local_lists[r] = (exit_idx_r, cont_idx_r) (local indices), offsets[r] =
    first global token of rank r.  Returns the global (exiting, continuing)
    stable partition."""
    ex, co = [], []
    for (e, c), (ne, nc), off in zip(local_lists, local_counts, offsets):
        ex.append(e[:ne] + off)
        co.append(c[:nc] + off)
    return torch.cat(ex), torch.cat(co)


def gather_rows(local: torch.Tensor, world: int, group=None, fill=0) -> torch.Tensor:
    """All-gather of per-rank row blocks [n_r, ...] with unequal n_r, in rank
    order: pad to the largest block, one all_gather_into_tensor, strip."""
    n_local = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.full((m,) + tuple(local.shape[1:]), fill, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * m: r * m + sizes[r]] for r in range(world)])


def gather_exit_layers(local_exit_layers: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """C1 for unequal shards: pad to the largest shard, all-gather, strip."""
    return gather_rows(local_exit_layers, world, group, fill=-1)


def label_shard(checkpoint_states: dict, final_states, tau: float, world: int, *, group=None,
                gather: bool = False, labeller=None) -> dict:
    """Calibration labelling token-sharded over the ranks (BASELINE config 4,
    ee/calibration.py:201-219): each rank labels its contiguous token shard in
    one labeller launch; the zero-norm count and the positives of every
    checkpoint are all-reduced; labels stay sharded (u8 [C, n_local]) unless
    gather=True (one all-gather, 1 B per token per checkpoint).

    `labeller(checkpoint_states, final_states, tau) -> (layers, sims [C, n],
    labels u8 [C, n], zero_counts [C])` defaults to the kernel
    (calibration.label_tensors); the CPU tests pass the oracle."""
    if labeller is None:
        from .calibration import label_tensors

        def labeller(cks, fin, t):
            return label_tensors(cks, fin, t, labels_dtype="u8")
    layers, sims, labels, zero = labeller(checkpoint_states, final_states, tau)
    counts = torch.stack([zero.to(torch.int64), labels.to(torch.int64).sum(dim=1)])
    dist.all_reduce(counts, group=group)
    out = {"layers": layers, "sims": sims, "labels": labels, "zero_counts": counts[0],
           "positives": counts[1]}
    if gather:
        out["global_labels"] = gather_rows(labels.t().contiguous(), world, group).t()
    return out
