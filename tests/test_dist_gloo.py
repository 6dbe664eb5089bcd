"""World-size-2 gloo tests (CPU) of the multi-GPU orchestration in paper_2001_00706_b200/dist.py.

The per-rank compute is the float64 oracle plugged in for the CUDA kernels, so what is tested is
the partitioning, the rank-order all-gather and the ordered fold -- the parts that NCCL runs in the
product path.  Rendezvous on 127.0.0.1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2001_00706_b200 import dist as sdist
from synth import brownian_paths


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_sig(x, depth):
    return torch.from_numpy(oracle.signature(x.numpy(), depth))


def _oracle_fold(sigs, C, depth):
    return torch.from_numpy(oracle.multi_combine(sigs.numpy(), C, depth))


def _oracle_combine_bwd(g, a, b, C, depth):
    return torch.from_numpy(np.stack([oracle.mul_vjp(g[i].numpy(), a[i].numpy(), b[i].numpy(), C, depth)[0]
                                      for i in range(g.shape[0])]))


def _oracle_local_bwd(g, x, out, depth, initial):
    gx, _, _ = oracle.signature_vjp_ex(g.numpy(), x.numpy(), depth,
                                       initial=None if initial is None else initial.numpy())
    return torch.from_numpy(gx)


def _work(rank, world, L, C, N):
    x = brownian_paths(2, L, C, seed=42)
    a, b = sdist.time_chunk_bounds(L, world, rank)
    xl = torch.from_numpy(x[:, a:b].astype(np.float64))
    sig, parts = sdist.dist_signature_timechunk(xl, N, local_sig=_oracle_sig, fold=_oracle_fold, return_parts=True)
    gsig = torch.from_numpy(np.random.default_rng(3).standard_normal(sig.shape))
    gx = sdist.dist_signature_timechunk_backward(gsig, xl, parts, N, fold=_oracle_fold,
                                                 combine_bwd=_oracle_combine_bwd, local_bwd=_oracle_local_bwd)
    # batch sharding: each rank its own slice, no collective
    lo, hi = sdist.batch_bounds(5, world, rank)
    xb = brownian_paths(5, 9, C, seed=7)
    sb = sdist.dist_signature_batch(torch.from_numpy(xb[lo:hi].astype(np.float64)), N, local_sig=_oracle_sig)
    return rank, sig.numpy(), lo, hi, sb.numpy(), gx


def _worker(rank, world, port, L, C, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put(_work(rank, world, L, C, N))
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put((rank, repr(e), None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L", [50, 51, 3])
def test_timechunk_and_batch_world2(L):
    C, N, world = 3, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, C, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for r in res:
        assert not isinstance(r[1], str), r[1]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = brownian_paths(2, L, C, seed=42)
    ref = oracle.signature(x, N)
    xb = brownian_paths(5, 9, C, seed=7)
    refb = oracle.signature(xb, N)
    for rank, sig, lo, hi, sb, _ in sorted(res, key=lambda r: r[0]):
        np.testing.assert_allclose(sig, ref, rtol=1e-11, atol=1e-13)  # replicated on every rank
        np.testing.assert_allclose(sb, refb[lo:hi], rtol=1e-12)
    # time-chunked backward: the ranks' point gradients, shared points summed, equal the VJP of the
    # whole path's signature
    gsig = np.random.default_rng(3).standard_normal(ref.shape)
    rg, _ = oracle.signature_vjp(gsig, x, N)
    got = sdist.assemble_timechunk_grad([r[5] for r in sorted(res, key=lambda r: r[0])], L).numpy()
    np.testing.assert_allclose(got, rg, rtol=1e-9, atol=1e-11)


def test_bounds_partition_exactly():
    for L in (2, 3, 10, 2 ** 22):
        for G in (1, 2, 4, 8):
            prev_end = 0
            for r in range(G):
                a, b = sdist.time_chunk_bounds(L, G, r)
                assert a == prev_end and b - 1 >= a
                prev_end = b - 1
            assert prev_end == L - 1
    for B in (1, 7, 1024):
        for G in (1, 2, 8):
            tot = sum(sdist.batch_bounds(B, G, r)[1] - sdist.batch_bounds(B, G, r)[0] for r in range(G))
            assert tot == B
