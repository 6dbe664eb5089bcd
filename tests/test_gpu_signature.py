"""GPU parity: the sm_100a signature forward/backward (through the C ABI) against the float64 oracle
on the same seeded float32 inputs.  Bars: 1e-4 (forward, per path and level) and 5e-4 (backward,
per path), BASELINE.json north_star; metric in tests/parity.py."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal, uniform_paths
from tests.parity import BWD_TOL, FWD_TOL, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu

sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


FWD_CASES = [
    # (C, N, B, L, kind)
    (4, 4, 32, 128, "brownian"),     # BASELINE config c1, full size
    (4, 4, 32, 128, "uniform"),
    (8, 5, 16, 128, "brownian"),     # c2 shape, subset of the batch
    (8, 5, 5, 37, "uniform"),
    (6, 4, 7, 100, "brownian"),      # c3 shape
    (4, 7, 6, 64, "brownian"),       # c4 shape
    (3, 6, 3, 333, "brownian"),      # c5 shape, short
    (2, 3, 9, 17, "uniform"),
    (1, 5, 4, 11, "monotone"),
    (5, 3, 13, 29, "uniform"),
    (7, 4, 3, 21, "brownian"),
    (8, 2, 70, 9, "uniform"),
    (3, 1, 5, 6, "brownian"),
    (2, 8, 3, 40, "brownian"),
    (4, 2, 1, 2, "uniform"),         # a single increment: exp(z)
]


def _paths(kind, B, L, C, seed):
    if kind == "monotone":  # no cancellation between increments (used for C = 1, R9)
        return np.cumsum(np.abs(brownian_paths(B, L, C, seed)), axis=1, dtype=np.float64).astype(np.float32)
    return brownian_paths(B, L, C, seed) if kind == "brownian" else uniform_paths(B, L, C, seed + 1000)


@pytest.mark.parametrize("C,N,B,L,kind", FWD_CASES)
def test_forward_parity(C, N, B, L, kind):
    x = _paths(kind, B, L, C, seed=C * 100 + N)
    got = sb.sig_signature(_cuda(x), N).cpu().numpy()
    ref = oracle.signature(x, N, threads=8)
    assert got.shape == ref.shape
    err = level_rel_err(got, ref, C, N)
    print(f"PARITY fwd C={C} N={N} B={B} L={L} {kind}: {err:.3e}")
    assert err < FWD_TOL, err


@pytest.mark.parametrize("C,N,B,L", [(6, 4, 5, 60), (4, 4, 3, 33), (8, 3, 4, 20), (3, 6, 2, 41),
                                     # many units per CTA in the staged stream kernel, odd S (rows
                                     # at every 4-byte phase), steps not a multiple of the image
                                     (5, 3, 700, 23), (2, 5, 1300, 14), (3, 2, 900, 3), (7, 3, 301, 40)])
def test_forward_stream_parity(C, N, B, L):
    x = brownian_paths(B, L, C, seed=7 + C)
    got = sb.sig_signature(_cuda(x), N, stream=True).cpu().numpy()
    ref = oracle.signature(x, N, stream=True, threads=8)
    assert got.shape == (B, L - 1, sum(C ** k for k in range(1, N + 1)))
    assert level_rel_err(got, ref, C, N, strict=True) < FWD_TOL  # strict: see tests/test_parity_floor.py


@pytest.mark.parametrize("bp", ["zero", "given"])
def test_forward_basepoint(bp):
    C, N, B, L = 4, 4, 6, 25
    x = brownian_paths(B, L, C, seed=3)
    bpv = normal((B, C), seed=4, scale=0.3)
    arg = True if bp == "zero" else _cuda(bpv)
    oarg = True if bp == "zero" else bpv
    got = sb.sig_signature(_cuda(x), N, basepoint=arg).cpu().numpy()
    ref = oracle.signature(x, N, basepoint=oarg)
    assert level_rel_err(got, ref, C, N) < FWD_TOL
    # a single point with a basepoint
    got1 = sb.sig_signature(_cuda(x[:, :1]), N, basepoint=arg).cpu().numpy()
    ref1 = oracle.signature(x[:, :1], N, basepoint=oarg)
    assert level_rel_err(got1, ref1, C, N) < FWD_TOL


def test_long_path_time_chunked():
    """One long path: the library splits it into time chunks and folds them with [x] in order."""
    C, N, L = 3, 6, 40000
    x = brownian_paths(1, L, C, seed=5)
    got = sb.sig_signature(_cuda(x), N).cpu().numpy()
    ref = oracle.signature(x, N)
    assert level_rel_err(got, ref, C, N) < FWD_TOL
    x2 = brownian_paths(3, 9001, 2, seed=6)  # ragged chunking, several paths
    got2 = sb.sig_signature(_cuda(x2), 5).cpu().numpy()
    assert level_rel_err(got2, oracle.signature(x2, 5, threads=3), 2, 5) < FWD_TOL


def test_empty_batch_and_determinism():
    x = brownian_paths(0, 10, 3, seed=1)
    assert sb.sig_signature(_cuda(x), 3).shape == (0, 39)
    y = _cuda(brownian_paths(64, 128, 8, seed=2))
    a = sb.sig_signature(y, 5)
    b = sb.sig_signature(y, 5)
    assert torch.equal(a, b)


BWD_CASES = [
    (4, 4, 16, 32, False),
    (8, 5, 8, 128, False),   # c2 shape
    (4, 7, 4, 64, False),    # c4 shape
    (3, 6, 3, 50, False),
    (2, 3, 5, 12, False),
    (1, 3, 2, 6, False),
    (5, 4, 3, 20, False),
    (6, 4, 2, 30, True),
    (4, 4, 3, 16, True),
    (8, 3, 4, 25, False),
    (3, 1, 4, 5, False),
    # more steps than one K2 tile (128): several gz flushes per path; B >= 148 keeps them unchunked
    (3, 6, 150, 300, False),
    (4, 4, 160, 700, False),
    (8, 5, 150, 200, False),
    (6, 4, 2, 300, True),
    # B just above one resident wave of one-CTA-per-SM kernels (a partial last wave)
    (4, 7, 150, 130, False),
    (8, 5, 158, 140, False),
]


@pytest.mark.parametrize("C,N,B,L,stream", BWD_CASES)
def test_backward_parity(C, N, B, L, stream):
    x = brownian_paths(B, L, C, seed=11 * C + N)
    S = sum(C ** k for k in range(1, N + 1))
    g = normal((B, L - 1, S) if stream else (B, S), seed=100 + C)
    xt = _cuda(x)
    out = sb.sig_signature(xt, N, stream=stream)
    gp, _ = sb.sig_signature_backward(_cuda(g), xt, out, N, stream=stream)
    ref, _ = oracle.signature_vjp(g, x, N, stream=stream, threads=8)
    err = path_rel_err(gp.cpu().numpy(), ref)
    print(f"PARITY bwd C={C} N={N} B={B} L={L} stream={stream}: {err:.3e}")
    assert err < BWD_TOL, err


def test_backward_basepoint_given_and_autograd():
    C, N, B, L = 4, 5, 4, 20
    x = brownian_paths(B, L, C, seed=21)
    bp = normal((B, C), seed=22, scale=0.2)
    g = normal((B, sum(C ** k for k in range(1, N + 1))), seed=23)
    xt = _cuda(x).requires_grad_(True)
    bpt = _cuda(bp).requires_grad_(True)
    out = sb.signature(xt, N, basepoint=bpt)
    out.backward(_cuda(g))
    rx, rb = oracle.signature_vjp(g, x, N, basepoint=bp)
    assert path_rel_err(xt.grad.cpu().numpy(), rx) < BWD_TOL
    assert path_rel_err(bpt.grad.cpu().numpy(), rb) < BWD_TOL


def test_paper_code_example():
    """signatory.signature(torch.rand(1, 10, 2), 4).sum().backward()."""
    torch.manual_seed(0)
    path = torch.rand(1, 10, 2, device="cuda", requires_grad=True)
    sig = sb.signature(path, 4)
    sig.sum().backward()
    x = path.detach().cpu().numpy()
    assert level_rel_err(sig.detach().cpu().numpy(), oracle.signature(x, 4), 2, 4) < FWD_TOL
    ref, _ = oracle.signature_vjp(np.ones((1, 30)), x, 4)
    assert path_rel_err(path.grad.cpu().numpy(), ref) < BWD_TOL


def test_c2_full_size_sampled():
    """BASELINE config c2 at full size (B=1024, L=128, C=8, N=5) in the launch configuration bench.py
    times: forward + backward of the whole batch, every 64th path checked against the oracle."""
    C, N, B, L = 8, 5, 1024, 128
    x = brownian_paths(B, L, C, seed=2)
    g = normal((B, 37448), seed=102)
    xt = _cuda(x)
    out = sb.sig_signature(xt, N)
    gp, _ = sb.sig_signature_backward(_cuda(g), xt, out, N)
    idx = np.arange(0, B, 64)
    ref = oracle.signature(x[idx], N, threads=16)
    ef = level_rel_err(out.cpu().numpy()[idx], ref, C, N)
    rg, _ = oracle.signature_vjp(g[idx], x[idx], N, threads=16)
    eb = path_rel_err(gp.cpu().numpy()[idx], rg)
    print(f"PARITY c2 full-size sampled: fwd {ef:.3e} bwd {eb:.3e}")
    assert ef < FWD_TOL and eb < BWD_TOL


def test_c3_full_size_sampled():
    """BASELINE config c3 at full size (B=256, L=1024, C=6, N=4, stream=True) in the launch
    configuration bench.py times (staged rows, TMA bulk stores): every 32nd path checked against the
    oracle at every step."""
    C, N, B, L = 6, 4, 256, 1024
    x = brownian_paths(B, L, C, seed=3)
    out = sb.sig_signature(_cuda(x), N, stream=True)
    idx = np.arange(5, B, 32)
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
    ref = oracle.signature(x[idx], N, stream=True, threads=16)
    err = level_rel_err(got, ref, C, N, strict=True)  # no floor (tests/test_parity_floor.py)
    print(f"PARITY c3 full-size sampled: {err:.3e}")
    assert err < FWD_TOL


@pytest.mark.parametrize("C,N", [(8, 2), (8, 3), (8, 4), (8, 5), (4, 6), (4, 7), (2, 11)])
@pytest.mark.parametrize("bp", [None, "zero", "given"])
def test_two_prefix_kernels(C, N, bp):
    """Shapes and batch sizes that take the two-prefix kernels (sig_fwd2_kernel: B >= 148, shapes
    (8,4), (8,5), (4,6), (4,7), (2,11); sig_bwd2_kernel: (8,2)..(8,5)), with every basepoint mode;
    every 16th path checked against the oracle."""
    B, L = 150, 23
    x = brownian_paths(B, L, C, seed=40 + N)
    S = sum(C ** k for k in range(1, N + 1))
    g = normal((B, S), seed=41 + N)
    bpa = normal((B, C), seed=42, scale=0.3) if bp == "given" else None
    xt = _cuda(x).requires_grad_(True)
    bpt = _cuda(bpa).requires_grad_(True) if bp == "given" else (True if bp == "zero" else None)
    out = sb.signature(xt, N, basepoint=bpt)
    out.backward(_cuda(g))
    idx = np.arange(0, B, 16)
    obp = bpa[idx] if bp == "given" else (True if bp == "zero" else None)
    ref = oracle.signature(x[idx], N, basepoint=obp, threads=8)
    assert level_rel_err(out.detach().cpu().numpy()[idx], ref, C, N) < FWD_TOL
    rx, rb = oracle.signature_vjp(g[idx], x[idx], N, basepoint=obp, threads=8)
    assert path_rel_err(xt.grad.cpu().numpy()[idx], rx) < BWD_TOL
    if bp == "given":
        assert path_rel_err(bpt.grad.cpu().numpy()[idx], rb) < BWD_TOL


def test_host_pipeline_matches_direct():
    """hostpipe.HostPipeline (host-resident batch in slices, copies overlapping the kernels) gives the
    same gradient as the direct calls, bit for bit, pass after pass."""
    from paper_2001_00706_b200.hostpipe import HostPipeline

    C, N, B, L = 8, 5, 300, 24
    x = brownian_paths(B, L, C, seed=61)
    g = normal((B, sum(C ** k for k in range(1, N + 1))), seed=62)
    xt, gt = _cuda(x), _cuda(g)
    ref, _ = sb.sig_signature_backward(gt, xt, sb.sig_signature(xt, N), N)
    xh = torch.from_numpy(x).pin_memory()
    gh = torch.from_numpy(g).pin_memory()
    out = torch.empty((B, L, C), dtype=torch.float32).pin_memory()
    pipe = HostPipeline([xh, gh], out, chunks=3)
    fn = lambda xd, gd: sb.sig_signature_backward(gd, xd, sb.sig_signature(xd, N), N)[0]  # noqa: E731
    for _ in range(2):
        pipe.run(fn)
        torch.cuda.synchronize()
        assert torch.equal(out, ref.cpu())


def test_c5_full_size():
    """BASELINE config c5 at full size: one path of L = 2^22 points, C = 3, N = 6, in the launch
    configuration bench.py times (time chunks folded in order).  The float64 oracle is run on 64
    time chunks in parallel (chunk j = points [j m, (j+1) m], sharing boundary points) and folded
    with its own [x] in time order -- Chen's identity, pinned by the oracle tests."""
    C, N, L = 3, 6, 2 ** 22
    x = brownian_paths(1, L, C, seed=5)
    got = sb.sig_signature(_cuda(x), N).cpu().numpy()
    nch = 64
    M = L - 1
    edges = [round(j * M / nch) for j in range(nch + 1)]
    m = max(b - a for a, b in zip(edges, edges[1:]))
    chunks = np.zeros((nch, m + 1, C), np.float32)
    for j, (a, b) in enumerate(zip(edges, edges[1:])):
        seg = x[0, a:b + 1]
        chunks[j, :len(seg)] = seg
        chunks[j, len(seg):] = seg[-1]  # repeated end point: a zero increment changes nothing
    sigs = oracle.signature(chunks, N, threads=16)
    ref = oracle.multi_combine(sigs[:, None, :], C, N)
    err = level_rel_err(got, ref.reshape(1, -1), C, N)
    print(f"PARITY c5 full-size: {err:.3e}")
    assert err < FWD_TOL


def test_fwd_bwd_host_entry_point():
    """sig_signature_fwd_bwd_host (host buffers in, host gradient out, slices whose copies overlap
    the kernels) equals the device calls bit for bit, for several slice counts incl. a ragged one,
    and pass after pass; also from pageable (non-pinned) host memory."""
    C, N, B, L = 8, 5, 301, 20
    x = brownian_paths(B, L, C, seed=71)
    g = normal((B, sum(C ** k for k in range(1, N + 1))), seed=72)
    xt, gt = _cuda(x), _cuda(g)
    ref, _ = sb.sig_signature_backward(gt, xt, sb.sig_signature(xt, N), N)
    ref = ref.cpu()
    xh = torch.from_numpy(x).pin_memory()
    gh = torch.from_numpy(g).pin_memory()
    for chunks in (1, 3, 4):
        for _ in range(2):
            out = sb.sig_signature_fwd_bwd_host(xh, gh, N, chunks=chunks)
            torch.cuda.synchronize()
            assert torch.equal(out, ref), chunks
    out = sb.sig_signature_fwd_bwd_host(torch.from_numpy(x), torch.from_numpy(g), N, chunks=2)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_c5_full_size_backward_sampled():
    """The c5 path (L = 2^22, C = 3, N = 6) through the reversible backward at full size, in the
    launch configuration of the library (time-parallel chunks), checked on sampled
    points: the float64 oracle computes the signatures of 256 time chunks (chunk j = points
    [e_j, e_{j+1}]), their ordered prefix products P_j and suffix products Q_j, and for three sampled
    chunks the gradient at the chunk's end (the left-operand VJP of P_{j+1} [x] Q_j at grad_out) and
    then the chunk's own VJP started from P_j (signature_vjp_ex with initial) -- the exact gradient
    of the chunk's interior points.
    Bars (R9, R21), 5e-4 each:
      * increment gradients dL/dz_t of every sampled chunk, per chunk (||.||inf / ||ref||inf): the
        GPU's are recovered exactly from its point gradients by a float64 prefix sum (dL/dz_t =
        -sum_{s<=t} dL/dx_s; each dL/dx_s was formed as a float32 difference of two dL/dz);
      * point gradients dL/dx per path (R9): normalised by the path's ||ref||inf, bounded below by
        the sampled chunks' values and the two end points' gradients (a stricter normaliser)."""
    from concurrent.futures import ThreadPoolExecutor

    C, N, L = 3, 6, 2 ** 22
    x = brownian_paths(1, L, C, seed=5)
    g = normal((1, oracle.sig_channels(C, N)), seed=105)
    xt = _cuda(x)
    gp, _ = sb.sig_signature_backward(_cuda(g), xt, sb.sig_signature(xt, N), N)
    gp = gp.cpu().numpy().astype(np.float64)
    gz_gpu = -np.cumsum(gp[0], axis=0)[:-1]  # [M, C]
    nch, M = 256, L - 1
    e = [round(j * M / nch) for j in range(nch + 1)]
    with ThreadPoolExecutor(16) as ex:  # the oracle's C calls release the GIL
        sigs = list(ex.map(lambda j: oracle.signature(x[:, e[j]:e[j + 1] + 1], N)[0], range(nch)))
    sigs = np.stack(sigs)
    refs = {}
    for j in (0, 137, nch - 1):
        P = oracle.multi_combine(sigs[:j, None], C, N)[0] if j > 0 else None
        Pn = oracle.multi_combine(sigs[:j + 1, None], C, N)[0]
        if j < nch - 1:
            Q = oracle.multi_combine(sigs[j + 1:, None], C, N)[0]
            gend = oracle.mul_vjp(g[0], Pn, Q, C, N)[0]
        else:
            gend = g[0].astype(np.float64)
        ref, _, _ = oracle.signature_vjp_ex(gend[None], x[:, e[j]:e[j + 1] + 1], N,
                                            initial=None if P is None else P[None])
        refs[j] = ref[0]
        gz_ref = -np.cumsum(ref[0], axis=0)[:-1]  # increments e_j .. e_{j+1}-1 (ref[0][0] = -dL/dz_{e_j})
        ez = float(np.max(np.abs(gz_gpu[e[j]:e[j + 1]] - gz_ref)) / np.max(np.abs(gz_ref)))
        print(f"PARITY c5 full-size backward, chunk {j}: increment gradient {ez:.3e}")
        assert ez < BWD_TOL, (j, ez)
    # the path's gradient norm: at least the sampled chunks' interior values and the end points
    # (dL/dx_0 = -dL/dz_0 and dL/dx_M = dL/dz_{M-1}, exact in the first / last chunk's VJP)
    den = max(max(float(np.max(np.abs(r))) for r in refs.values()),
              float(np.max(np.abs(refs[0][0]))), float(np.max(np.abs(refs[nch - 1][-1]))))
    for j, r in refs.items():
        a, b = e[j] + 1, e[j + 1]  # interior points only (boundary points get shares of two chunks)
        ex_ = float(np.max(np.abs(gp[0, a:b] - r[1:-1]))) / den
        print(f"PARITY c5 full-size backward, chunk {j}: point gradient (per path, R9) {ex_:.3e}")
        assert ex_ < BWD_TOL, (j, ex_)
    assert float(np.max(np.abs(gp[0, 0] - refs[0][0]))) / den < BWD_TOL
    assert float(np.max(np.abs(gp[0, -1] - refs[nch - 1][-1]))) / den < BWD_TOL
