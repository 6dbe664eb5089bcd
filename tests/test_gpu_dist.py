"""World-size-2 test of the multi-GPU path with the REAL kernels (paper_2001_00706_b200/dist.py).

This round's boxes have one GPU, so both ranks share cuda:0 over a gloo group; dist.py stages the
[G, S] exchange through host memory in that case (with NCCL on a multi-GPU box it gathers the
device tensors in place).  Everything else is the product path: the time-chunked signature (local
K1 + in-GPU fold, all-gather in rank = time order, ordered fold), its time-chunked backward (chunk-end
gradients from the gathered chunk signatures, local reversible backward started at the prefix
product), and batch sharding -- checked against the float64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, C, N, q):
    import torch.distributed as dist

    import paper_2001_00706_b200 as sb
    from paper_2001_00706_b200 import dist as sdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        x = brownian_paths(1, L, C, seed=5)
        a, b = sdist.time_chunk_bounds(L, world, rank)
        xl = torch.from_numpy(np.ascontiguousarray(x[:, a:b])).cuda()
        sig, parts = sdist.dist_signature_timechunk(xl, N, return_parts=True)
        gsig = torch.from_numpy(normal(tuple(sig.shape), seed=55)).cuda()
        gx = sdist.dist_signature_timechunk_backward(gsig, xl, parts, N)
        # batch sharding of a c2-shaped batch: each rank its own paths, forward + backward
        xb = brownian_paths(12, 40, 8, seed=2)
        lo, hi = sdist.batch_bounds(12, world, rank)
        xbl = torch.from_numpy(np.ascontiguousarray(xb[lo:hi])).cuda()
        sbl = sdist.dist_signature_batch(xbl, 5)
        gb = torch.from_numpy(normal((12, sb.sig_signature_channels(8, 5)), seed=6)[lo:hi]).cuda()
        gpb, _ = sb.sig_signature_backward(gb, xbl, sbl, 5)
        torch.cuda.synchronize()
        q.put((rank, sig.cpu().numpy(), gx.cpu().numpy(), lo, hi, sbl.cpu().numpy(), gpb.cpu().numpy()))
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put((rank, repr(e), None, None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L", [20001, 4097])
def test_world2_timechunk_and_batch_real_kernels(L):
    C, N, world = 3, 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, C, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert not isinstance(r[1], str), r[1]
    x = brownian_paths(1, L, C, seed=5)
    ref = oracle.signature(x, N)
    for r in res:  # replicated on every rank
        e = level_rel_err(r[1], ref, C, N)
        print(f"PARITY dist timechunk fwd L={L} rank {r[0]}: {e:.3e}")
        assert e < FWD_TOL, e
    gsig = normal((1, oracle.sig_channels(C, N)), seed=55)
    rg, _ = oracle.signature_vjp(gsig, x, N)
    from paper_2001_00706_b200 import dist as sdist

    got = sdist.assemble_timechunk_grad([torch.from_numpy(r[2]) for r in res], L).numpy()
    e = path_rel_err(got, rg)
    print(f"PARITY dist timechunk bwd L={L}: {e:.3e}")
    assert e < BWD_TOL, e
    xb = brownian_paths(12, 40, 8, seed=2)
    refb = oracle.signature(xb, 5, threads=8)
    gb = normal((12, oracle.sig_channels(8, 5)), seed=6)
    rgb, _ = oracle.signature_vjp(gb, xb, 5, threads=8)
    for r in res:
        lo, hi = r[3], r[4]
        assert level_rel_err(r[5], refb[lo:hi], 8, 5) < FWD_TOL
        assert path_rel_err(r[6], rgb[lo:hi]) < BWD_TOL
