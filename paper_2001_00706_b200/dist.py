"""Multi-GPU composition of the hot path over one box (one process per GPU, torch.distributed).

Two ways to partition ("naive parallelism over the batch dimension" and "splitting the
computation up into chunks" of the noncommutative reduction):

* Batch sharding -- the paths are independent, so rank r simply processes its own slice
  [r*B/G, (r+1)*B/G) of the batch (``batch_bounds``).  There is no collective on the data path
  (path gradients are per sample).
* Time chunking (one very long path, BASELINE config c5) -- rank r owns the points
  [r*M/G, (r+1)*M/G] (M = L-1 increments; consecutive chunks share their boundary point, so the
  increments are partitioned exactly, reading R16).  Each rank computes its chunk signature S_r on
  its GPU (the library itself splits the chunk again over the SMs and folds), the G signatures are
  exchanged with ONE ``all_gather_into_tensor`` (rank order = time order), and every rank folds
  them in time order with the group-like product (Chen's identity, eq-grouplike P:L84-87) --
  the result is replicated, no broadcast needed.  The message is G*S floats (c5: 4.4 KB per rank),
  latency-bound over NVLink/NVSwitch.
* Time-chunked backward (SURVEY 8(f)1 across ranks) -- with Sig = P_r [x] S_r [x] Q_r
  (P_r the product of the earlier chunks, Q_r of the later ones, both from the same all-gather), the
  gradient at the end of rank r's chunk is the left-operand VJP of (P_r [x] S_r) [x] Q_r, and the
  rank reverses its own chunk from there, starting at P_r (the ``initial`` option): one all-gather,
  no further exchange.  A point shared by ranks r and r+1 receives a share from each
  (``assemble_timechunk_grad`` adds them).

The compute steps are pluggable so that the orchestration -- bounds, ordering, the exchange -- is
covered by world-size-2 gloo tests on CPU with the float64 oracle; in the product path they are the
CUDA kernels of libsig.so and the exchange is NCCL over NVLink.  With a gloo group and CUDA tensors
(two ranks sharing one GPU in the GPU tests) the exchange is staged through host memory.
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


def _sig_channels(C: int, depth: int) -> int:
    return sum(C ** k for k in range(1, depth + 1))


def _default_local_sig(x: torch.Tensor, depth: int) -> torch.Tensor:
    import paper_2001_00706_b200 as sb

    return sb.sig_signature(x, depth)


def _default_fold(sigs: torch.Tensor, C: int, depth: int) -> torch.Tensor:
    import paper_2001_00706_b200 as sb

    return sb.sig_multi_signature_combine(sigs, C, depth)


def _default_combine_bwd(g: torch.Tensor, a: torch.Tensor, b: torch.Tensor, C: int, depth: int):
    import paper_2001_00706_b200 as sb

    return sb.sig_signature_combine_backward(g, a, b, C, depth)[0]


def _default_local_bwd(g: torch.Tensor, x: torch.Tensor, out: torch.Tensor, depth: int,
                       initial: Optional[torch.Tensor]) -> torch.Tensor:
    import paper_2001_00706_b200 as sb

    gp, _, _ = sb.sig_signature_backward_ex(g, x, out, depth, initial=initial, want_grad_initial=False)
    return gp


def _all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """[world, *t.shape] in rank order.  NCCL gathers device tensors in place; a gloo group with a
    CUDA tensor (several ranks on one GPU in tests) is staged through host memory."""
    world = dist.get_world_size(group)
    stage = t.is_cuda and dist.get_backend(group) == "gloo"
    src = t.detach().reshape(-1).contiguous()
    if stage:
        src = src.cpu()
    flat = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(flat, src, group=group)
    if stage:
        flat = flat.to(t.device)
    return flat.view((world,) + tuple(t.shape))


def _local_chunk_sig(x_local, depth, local_sig):
    B, Lr, C = x_local.shape
    if Lr >= 2:
        return local_sig(x_local, depth).contiguous()
    # no increment on this rank (more ranks than increments): the group identity
    return torch.zeros((B, _sig_channels(C, depth)), dtype=x_local.dtype, device=x_local.device)


def dist_signature_timechunk(x_local: torch.Tensor, depth: int, group=None,
                             local_sig: Optional[Callable] = None, fold: Optional[Callable] = None,
                             return_parts: bool = False):
    """Signature of one long path split in time over the ranks of ``group``.

    x_local: [B, L_r, C] -- this rank's points (time_chunk_bounds), on this rank's device.
    Returns the signature of the whole path, [B, S], on every rank (and the gathered chunk
    signatures [G, B, S] with return_parts=True, as the backward needs them).
    """
    local_sig = local_sig or _default_local_sig
    fold = fold or _default_fold
    world = dist.get_world_size(group)
    C = x_local.shape[2]
    s_local = _local_chunk_sig(x_local, depth, local_sig)
    if world == 1:
        return (s_local, s_local.unsqueeze(0)) if return_parts else s_local
    parts = _all_gather_rows(s_local, group)  # rank order == time order
    sig = fold(parts, C, depth)
    return (sig, parts) if return_parts else sig


def dist_signature_timechunk_backward(grad_sig: torch.Tensor, x_local: torch.Tensor, parts: torch.Tensor, depth: int,
                                      group=None, fold: Optional[Callable] = None,
                                      combine_bwd: Optional[Callable] = None,
                                      local_bwd: Optional[Callable] = None) -> torch.Tensor:
    """Gradient w.r.t. this rank's points [B, L_r, C] of a loss whose gradient w.r.t. the whole
    path's signature is grad_sig [B, S] (the same on every rank); parts = the gathered chunk
    signatures of the forward.  No collective: everything needed came with the forward's
    all-gather.  Shared boundary points get one share per rank (assemble_timechunk_grad)."""
    fold = fold or _default_fold
    combine_bwd = combine_bwd or _default_combine_bwd
    local_bwd = local_bwd or _default_local_bwd
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, Lr, C = x_local.shape
    if Lr < 2:
        return torch.zeros_like(x_local)
    prefix = fold(parts[:rank], C, depth) if rank > 0 else None          # P_r
    upto = fold(parts[:rank + 1], C, depth) if rank > 0 else parts[0]      # P_{r+1} = P_r [x] S_r
    if rank < world - 1:
        suffix = fold(parts[rank + 1:], C, depth) if rank < world - 2 else parts[world - 1]  # Q_r
        g_end = combine_bwd(grad_sig.contiguous(), upto.contiguous(), suffix.contiguous(), C, depth)
    else:
        g_end = grad_sig
    return local_bwd(g_end.contiguous(), x_local, upto.contiguous(), depth,
                     None if prefix is None else prefix.contiguous())


def assemble_timechunk_grad(local_grads, L: int) -> torch.Tensor:
    """Sum the ranks' point gradients (list in rank order, each [B, L_r, C]) into [B, L, C]."""
    world = len(local_grads)
    B, _, C = local_grads[0].shape
    out = torch.zeros((B, L, C), dtype=local_grads[0].dtype, device=local_grads[0].device)
    for r, g in enumerate(local_grads):
        a, b = time_chunk_bounds(L, world, r)
        out[:, a:b] += g
    return out


def dist_signature_batch(x_local: torch.Tensor, depth: int, local_sig: Optional[Callable] = None) -> torch.Tensor:
    """Batch-sharded forward: each rank transforms its own paths; no collective."""
    return (local_sig or _default_local_sig)(x_local, depth)
