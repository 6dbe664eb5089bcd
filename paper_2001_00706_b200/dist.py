"""Multi-GPU composition of the hot path over one box (one process per GPU, torch.distributed).

Two ways to partition ("naive parallelism over the batch dimension" and "splitting the
computation up into chunks" of the noncommutative reduction):

* Batch sharding -- the paths are independent, so rank r simply processes its own slice
  [r*B/G, (r+1)*B/G) of the batch (``batch_bounds``).  There is no collective on the data path
  (path gradients are per sample).
* Time chunking (one very long path, BASELINE config c5) -- rank r owns the points
  [r*M/G, (r+1)*M/G] (M = L-1 increments; consecutive chunks share their boundary point, so the
  increments are partitioned exactly, reading R16).  Each rank computes its chunk signature on
  its GPU (the library itself splits the chunk again over the SMs and folds), the G signatures are
  exchanged with ONE ``all_gather_into_tensor`` (rank order = time order), and every rank folds
  them in time order with the group-like product (Chen's identity, eq-grouplike P:L84-87) --
  the result is replicated, no broadcast needed.  The message is G*S floats (c5: 4.4 KB per rank),
  latency-bound over NVLink/NVSwitch.

The compute steps are pluggable (``local_sig`` / ``fold``) so that the orchestration -- bounds,
ordering, the exchange -- is covered by world-size-2 gloo tests on CPU; in the product path they
are the CUDA kernels of libsig.so (sig_signature, sig_multi_signature_combine) and the exchange is
NCCL over NVLink.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def batch_bounds(B: int, world: int, rank: int) -> tuple[int, int]:
    """Rank r's slice of a batch of B paths: [r*B//G, (r+1)*B//G)."""
    return rank * B // world, (rank + 1) * B // world


def time_chunk_bounds(L: int, world: int, rank: int) -> tuple[int, int]:
    """Point range [start, stop) of rank r for a path of L points (M = L-1 increments): the
    increments [r*M//G, (r+1)*M//G) i.e. points r*M//G .. (r+1)*M//G inclusive."""
    M = L - 1
    a, b = rank * M // world, (rank + 1) * M // world
    return a, b + 1


def _default_local_sig(x: torch.Tensor, depth: int) -> torch.Tensor:
    import paper_2001_00706_b200 as sb

    return sb.sig_signature(x, depth)


def _default_fold(sigs: torch.Tensor, C: int, depth: int) -> torch.Tensor:
    import paper_2001_00706_b200 as sb

    return sb.sig_multi_signature_combine(sigs, C, depth)


def dist_signature_timechunk(x_local: torch.Tensor, depth: int, group=None,
                             local_sig: Optional[Callable] = None, fold: Optional[Callable] = None) -> torch.Tensor:
    """Signature of one long path split in time over the ranks of ``group``.

    x_local: [B, L_r, C] -- this rank's points (time_chunk_bounds), on this rank's device.
    Returns the signature of the whole path, [B, S], on every rank.
    """
    local_sig = local_sig or _default_local_sig
    fold = fold or _default_fold
    world = dist.get_world_size(group)
    B, _, C = x_local.shape
    if x_local.shape[1] >= 2:
        s_local = local_sig(x_local, depth).contiguous()  # [B, S]
    else:  # no increment on this rank (more ranks than increments): the group identity
        S = sum(C ** k for k in range(1, depth + 1))
        s_local = torch.zeros((B, S), dtype=x_local.dtype, device=x_local.device)
    if world == 1:
        return s_local
    flat = torch.empty(world * s_local.numel(), dtype=s_local.dtype, device=s_local.device)
    dist.all_gather_into_tensor(flat, s_local.reshape(-1), group=group)  # rank order == time order
    return fold(flat.view((world,) + tuple(s_local.shape)), C, depth)


def dist_signature_batch(x_local: torch.Tensor, depth: int, local_sig: Optional[Callable] = None) -> torch.Tensor:
    """Batch-sharded forward: each rank transforms its own paths; no collective."""
    return (local_sig or _default_local_sig)(x_local, depth)
