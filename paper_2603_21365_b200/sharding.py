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
    """Preallocated C1/C2 all-gathers for equal shards of n_local tokens."""

    def __init__(self, n_local: int, world: int, device, exit_map_dtype=torch.uint8, group=None):
        self.n_local = n_local
        self.world = world
        self.group = group
        self.exit_map = torch.empty(world * n_local, dtype=exit_map_dtype, device=device)
        self.counts = torch.empty(world * 2, dtype=torch.int64, device=device)
        self.indices = torch.empty(world * n_local, dtype=torch.int64, device=device)

    def all_gather(self, local_exit_map, local_exit_idx, local_counts, rank=None):
        dist.all_gather_into_tensor(self.exit_map, local_exit_map.contiguous(), group=self.group)
        dist.all_gather_into_tensor(self.counts, local_counts.contiguous(), group=self.group)
        dist.all_gather_into_tensor(self.indices, local_exit_idx.contiguous(), group=self.group)

    def global_exit_indices(self) -> torch.Tensor:
        """Concatenate the per-rank stable exit lists with rank offsets (C2)."""
        parts = []
        counts = self.counts.view(self.world, 2).cpu()
        for r in range(self.world):
            k = int(counts[r, 0])
            seg = self.indices[r * self.n_local: r * self.n_local + k]
            parts.append(seg + r * self.n_local)
        return torch.cat(parts) if parts else self.indices[:0]


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


def gather_exit_layers(local_exit_layers: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """C1 for unequal shards: pad to the largest shard, all-gather, strip."""
    n_local = torch.tensor([local_exit_layers.numel()], dtype=torch.int64,
                           device=local_exit_layers.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.full((m,), -1, dtype=local_exit_layers.dtype, device=local_exit_layers.device)
    pad[: local_exit_layers.numel()] = local_exit_layers
    out = torch.empty(world * m, dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * m: r * m + sizes[r]] for r in range(world)])
