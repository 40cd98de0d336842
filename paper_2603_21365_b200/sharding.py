"""Token sharding across the GPUs of one box.

Every per-token quantity on this path is row-independent, so rank r owns the
contiguous token range shard_range(n, r, R) and runs the kernels on it with no
exchange during compute.  The only collectives are

  C1  all-gather of the per-token exit map, 1 byte per token (the u8 mask,
      or u8 exit codes layer + 1 for a multi-checkpoint selection), and
  C2  the global compacted exit indices, derived LOCALLY on every rank by
      one stable compaction scan of the gathered map — because shards are
      contiguous and in rank order, the gathered map is the global map and
      its stable partition is bit-identical to the single-GPU result by
      construction.  No index list crosses NVLink (ExitMapGather).
      `assemble_partition` keeps the host-side concatenation of per-rank
      lists (rank offsets added) for callers that hold them anyway.

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
    """C1 + C2 as ONE all-gather of 1 byte per token, for equal shards of
    n_local tokens.

    Each rank's send buffer is its shard's u8 exit map: the route kernel's
    mask (1 = exited) written straight into `exit_map`, or for a multi-
    checkpoint selection the exit codes `encode(exit_layers)` (layer + 1,
    0 = NO_EXIT).  After the all-gather, `recv` IS the global exit map in
    token order (shards are contiguous and in rank order), and every rank
    derives C2 locally with one compaction scan of it (`global_exit_indices`,
    bit-identical to the single-GPU stable partition by construction).  The
    rank's own stable partition stays local (the fused kernel's outputs).
    Against gathering int64 index lists this is 9x fewer bytes per token on
    the wire.

    `compactor(mask_u8, out_idx, counts)` and the codec default to the
    kernels (tide_compact / tide_exit_encode / tide_exit_decode); the CPU
    host-logic tests pass the oracle."""

    def __init__(self, n_local: int, world: int, device, group=None, *, compactor=None):
        self.n_local = n_local
        self.world = world
        self.group = group
        self.device = torch.device(device)
        self.send = torch.zeros(n_local, dtype=torch.uint8, device=self.device)
        self.recv = torch.zeros(world * n_local, dtype=torch.uint8, device=self.device)
        self.exit_map = self.send
        self.global_idx = torch.empty(world * n_local, dtype=torch.int64, device=self.device)
        self.global_counts = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._compactor = compactor
        # gloo has no CUDA all-gather: stage through host buffers (the one-GPU
        # multi-rank tests); NCCL gathers device memory directly
        self._single = world == 1  # one rank: the gathered map is the send buffer
        if not self._single and not dist.is_initialized():
            raise RuntimeError(f"ExitMapGather over {world} ranks needs an initialised "
                               f"process group")
        self._staged = (not self._single and self.device.type == "cuda"
                        and dist.get_backend(group) == dist.Backend.GLOO)
        if self._staged:
            self._hsend = torch.empty(n_local, dtype=torch.uint8)
            self._hrecv = torch.empty(world * n_local, dtype=torch.uint8)

    @property
    def nbytes(self) -> int:
        """Bytes each rank contributes to the collective."""
        return self.n_local

    def encode(self, exit_layers: torch.Tensor) -> None:
        """Write a shard's int64 exit map (NO_EXIT = -1) as u8 codes into the
        send buffer (one kernel; layers must be < 255)."""
        if exit_layers.numel() != self.n_local:
            raise ValueError(f"exit map has {exit_layers.numel()} tokens, shard has "
                             f"{self.n_local}")
        if self.device.type == "cuda":
            from . import _device as D
            from . import _native as N
            N.check(N.load().tide_exit_encode(exit_layers.data_ptr(), self.n_local,
                                              self.send.data_ptr(),
                                              D.stream_handle(self.device)), "tide_exit_encode")
        else:
            self.send.copy_((exit_layers + 1).to(torch.uint8))

    def all_gather(self, async_op: bool = False):
        if self._single:
            self.recv.copy_(self.send)
            return None
        if self._staged:
            self._hsend.copy_(self.send)
            dist.all_gather_into_tensor(self._hrecv, self._hsend, group=self.group)
            self.recv.copy_(self._hrecv)
            return None
        return dist.all_gather_into_tensor(self.recv, self.send, group=self.group,
                                           async_op=async_op)

    def global_exit_map(self) -> torch.Tensor:
        """C1: the exit map (mask or codes) of all ranks' shards, in token order."""
        return self.recv

    def global_exit_layers(self) -> torch.Tensor:
        """C1 for exit codes: the global int64 exit map (NO_EXIT = -1)."""
        out = torch.empty(self.world * self.n_local, dtype=torch.int64, device=self.device)
        if self.device.type == "cuda":
            from . import _device as D
            from . import _native as N
            N.check(N.load().tide_exit_decode(self.recv.data_ptr(), out.numel(), out.data_ptr(),
                                              D.stream_handle(self.device)), "tide_exit_decode")
        else:
            out.copy_(self.recv.to(torch.int64) - 1)
        return out

    def global_exit_indices(self, sync: bool = True):
        """C2, derived locally: one stable compaction scan of the gathered
        map.  Returns the global exit indices (a view of `global_idx`) when
        `sync`, else None with the count left in `global_counts[0]` on the
        device (no host round trip; the bench's step)."""
        n = self.world * self.n_local
        if self._compactor is not None:
            self._compactor(self.recv, self.global_idx, self.global_counts)
        else:
            from . import _device as D
            from . import _native as N
            N.check(N.load().tide_compact(self.recv.data_ptr(), n, None, None, 0, None, 0, 0, 0,
                                          self.global_idx.data_ptr(), None, None, None,
                                          self.global_counts.data_ptr(),
                                          D.workspace(self.device).data_ptr(),
                                          D.stream_handle(self.device)), "tide_compact")
        if not sync:
            return None
        return self.global_idx[: int(self.global_counts[0])]


def select_exits_shard(hidden_states, bank, config, gather: ExitMapGather, *,
                       selector=None) -> torch.Tensor:
    """Token-sharded exit selection (BASELINE config 5, ee/runtime.py:151-178):
    this rank's captures hold its contiguous token shard; the local exit map
    comes from one select_exits call (peeling chain / decode kernel, no
    exchange during compute), is written as u8 codes into the gather's send
    buffer and all-gathered (C1).  Returns the local int64 exit map; the
    global map / exit indices are then `gather.global_exit_layers()` and
    `gather.global_exit_indices()` (C2, derived locally).

    `selector(hidden_states, bank, config) -> int64 [n_local]` defaults to
    runtime.select_exits; the CPU tests pass the oracle."""
    if selector is None:
        from .runtime import select_exits as selector
    if bank.num_layers >= 255:
        raise ValueError("u8 exit codes hold layers < 255; use gather_exit_layers")
    local = selector(hidden_states, bank, config)
    gather.encode(local)
    gather.all_gather()
    return local


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
    if world > 1:
        dist.all_reduce(counts, group=group)
    out = {"layers": layers, "sims": sims, "labels": labels, "zero_counts": counts[0],
           "positives": counts[1]}
    if gather:
        out["global_labels"] = gather_rows(labels.t().contiguous(), world, group).t()
    return out
