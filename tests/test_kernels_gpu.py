"""Single-kernel numerics: each sm_100a kernel against a plain torch fp32 reference
of the same op (the kernels' own contract, independent of the EL bookkeeping)."""
import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _testing_lib():
    from paper_2105_04779_b200 import capi

    L = capi.lib()
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.elattn_gpu_testing_gemm_bf16.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64,
                                               i32, i32, i32, i32, ctypes.c_float, i32, vp]
    L.elattn_gpu_testing_decode_bf16.argtypes = [vp, vp, vp, i32, i32, i32, i32, ctypes.c_float, vp, i32, vp]
    return L, capi


def gemm_case(kernel, M, N, K, Z, layout, seed=0, with_bias=True, alpha=1.0):
    """layout: 'plain' (A [Z][M][K], B [Z][N][K]) or 'heads' (A columns of a [M][Z*K]
    matrix, C rows r*Z+z of a [M*Z][N] matrix — the query-expansion pattern)."""
    import torch

    L, capi = _testing_lib()
    g = torch.Generator(device="cuda").manual_seed(seed)
    bf = torch.bfloat16
    if layout == "plain":
        A = torch.randn(Z, M, K, generator=g, device="cuda").to(bf)
        lda, sAz = K, M * K
        Aview = A.float()
        Cbuf = torch.zeros(Z, M, N, device="cuda", dtype=bf)
        ldc, sCz = N, M * N
    else:
        Afull = torch.randn(M, Z * K, generator=g, device="cuda").to(bf)
        A = Afull
        lda, sAz = Z * K, K
        Aview = Afull.float().view(M, Z, K).permute(1, 0, 2)
        Cbuf = torch.zeros(M * Z, N, device="cuda", dtype=bf)
        ldc, sCz = Z * N, N
    Bm = torch.randn(Z, N, K, generator=g, device="cuda").to(bf)
    bias = torch.randn(Z, N, generator=g, device="cuda") if with_bias else None
    rc = L.elattn_gpu_testing_gemm_bf16(A.data_ptr(), lda, sAz, Bm.data_ptr(), K, N * K, Cbuf.data_ptr(), ldc, sCz,
                                        bias.data_ptr() if bias is not None else None, N, M, N, K, Z, alpha, kernel,
                                        torch.cuda.current_stream().cuda_stream)
    capi.check(rc)
    torch.cuda.synchronize()
    want = alpha * torch.einsum("zmk,znk->zmn", Aview, Bm.float())
    if bias is not None:
        want = want + bias[:, None, :]
    got = Cbuf.float().view(M, Z, N).permute(1, 0, 2) if layout == "heads" else Cbuf.float()
    return got, want


@pytest.mark.parametrize("kernel", [1, 0])
@pytest.mark.parametrize("M,N,K,Z,layout", [
    (128, 128, 64, 1, "plain"),
    (256, 1024, 1024, 1, "plain"),      # Q = Y.W_Q (BART)
    (200, 64, 1024, 3, "plain"),        # M tail, N = d_k
    (1280, 1024, 64, 16, "heads"),      # q'_{r,i} = Q_{r,i}.W_K,i^T (BART, B=320)
    (77, 96, 128, 2, "heads"),
])
def test_gemm_vs_torch(kernel, M, N, K, Z, layout):
    got, want = gemm_case(kernel, M, N, K, Z, layout, seed=M + N + K)
    err = (got - want).abs().max().item() / want.abs().max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("bn,mt,kbp", [
    (64, 1, 1), (64, 2, 1), (64, 1, 2), (64, 2, 2),
    (128, 1, 1), (128, 2, 1), (128, 1, 2), (128, 2, 2),
    (256, 1, 1), (256, 1, 2),
])
@pytest.mark.parametrize("M,N,K,Z,layout", [
    (1280, 1024, 1024, 1, "plain"),     # Q = Y.W_Q / out = V.W_O (BART, B = 320)
    (300, 64, 1024, 16, "heads"),       # V_i = C_i.W_V,i shape class, M tail
    (1280, 1024, 64, 16, "heads"),      # q' expansion (BART, B = 320)
    (77, 192, 128, 3, "plain"),         # M and N tails
    (140, 128, 192, 2, "heads"),        # K / 64 odd: the last 2-k-block box runs past K
])
def test_gemm_block_shapes(bn, mt, kbp, M, N, K, Z, layout):
    """Every instantiation of the tcgen05 GEMM family (tile width, m-subtiles sharing the B
    slice, k-blocks per TMA box) against torch fp32, including M / N / K tails."""
    L, capi = _testing_lib()
    L.elattn_gpu_testing_gemm_config.argtypes = [ctypes.c_int] * 3
    capi.check(L.elattn_gpu_testing_gemm_config(bn, mt, kbp))
    try:
        for tma in (0, 1):  # both epilogues: coalesced st.global / 128-row TMA stores
            capi.check(L.elattn_gpu_testing_gemm_epilogue(tma))
            got, want = gemm_case(1, M, N, K, Z, layout, seed=M + N + K + bn + mt + kbp, alpha=0.5)
            err = (got - want).abs().max().item() / want.abs().max().item()
            assert err < 1e-2, (tma, err)
    finally:
        capi.check(L.elattn_gpu_testing_gemm_config(0, 0, 0))
        capi.check(L.elattn_gpu_testing_gemm_epilogue(-1))


@pytest.mark.parametrize("sk", [0, 2, 4, 8])
@pytest.mark.parametrize("M,N,K,Z,layout", [
    (128, 1024, 1024, 1, "plain"),      # Q = Y.W_Q / out = V.W_O at B = 32 (beam 4)
    (128, 64, 1024, 16, "heads"),       # V_i = C_i.W_V,i at B = 32 (head-strided A and C)
    (77, 192, 512, 3, "plain"),         # M and N tails
    (256, 128, 1024, 2, "heads"),       # two m-tiles
])
def test_gemm_splitk(sk, M, N, K, Z, layout):
    """The small-M split-K GEMM (cluster of sk CTAs per 128 x 64 tile, DSMEM reduce-scatter
    of the partial accumulators) against torch fp32, against the plain tile kernel
    (sk = 0), and bit-reproducible across runs (rank-ordered reduction)."""
    L, capi = _testing_lib()
    L.elattn_gpu_testing_gemm_splitk.argtypes = [ctypes.c_int]
    capi.check(L.elattn_gpu_testing_gemm_splitk(sk))
    try:
        got, want = gemm_case(1, M, N, K, Z, layout, seed=M + N + K + sk, alpha=0.5)
        err = (got - want).abs().max().item() / want.abs().max().item()
        assert err < 1e-2, err
        again, _ = gemm_case(1, M, N, K, Z, layout, seed=M + N + K + sk, alpha=0.5)
        assert (again == got).all()
    finally:
        capi.check(L.elattn_gpu_testing_gemm_splitk(-1))


def decode_ref(qp, H, rows, scale, npi=None):
    """torch fp32: C[b*rows+q] = softmax(q' H_b^T * scale) H_b."""
    import torch

    B, n, d_m = H.shape
    q = qp.float().view(B, rows, d_m)
    Hf = H.float()
    S = torch.einsum("bqd,bnd->bqn", q, Hf) * scale
    if npi is not None:
        mask = torch.arange(n, device=H.device)[None, None, :] >= npi.view(B, 1, 1)
        S = S.masked_fill(mask, float("-inf"))
        Hf = Hf.masked_fill((torch.arange(n, device=H.device)[None, :, None] >= npi.view(B, 1, 1)), 0.0)
    P = torch.softmax(S, dim=-1)
    return torch.einsum("bqn,bnd->bqd", P, Hf).reshape(B * rows, d_m)


@pytest.mark.parametrize("kernel", [1, 0])
@pytest.mark.parametrize("B,rows,n,d_m", [
    (1, 64, 32, 512), (2, 64, 1024, 1024), (3, 16, 77, 1024), (2, 48, 300, 256), (5, 64, 129, 768),
    (2, 128, 300, 1024), (3, 192, 1024, 512), (80, 192, 256, 1024),  # beam 8 / 12: virtual inputs
    (2, 80, 300, 1024), (3, 96, 129, 512), (5, 160, 257, 1024),      # beam 5 / 6 / 10: partial virtual inputs
])
def test_decode_vs_torch(kernel, B, rows, n, d_m):
    import torch

    L, capi = _testing_lib()
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + n)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    ctx = torch.full((B * rows, d_m), float("nan"), device="cuda", dtype=torch.bfloat16)
    scale = 1.0 / 8.0
    capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, scale,
                                                ctx.data_ptr(), kernel, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = decode_ref(qp, H, rows, scale)
    err = (ctx.float() - want).abs().max().item() / want.abs().max().item()
    assert torch.isfinite(ctx.float()).all()
    assert err < 2e-2, err


@pytest.mark.parametrize("kernel", [1, 0])
def test_decode_large_scores_rescale_path(kernel):
    """Scores whose running max jumps by far more than 2^8 between tiles force the
    lazy O rescale (FA4-style threshold) — must stay exact."""
    import torch

    L, capi = _testing_lib()
    B, rows, n, d_m = 2, 64, 256, 512
    g = torch.Generator(device="cuda").manual_seed(7)
    qp = torch.randn(B * rows, d_m, generator=g, device="cuda").to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1)
    H[:, 100:] *= 4.0  # later tiles dominate: max grows tile after tile
    H = H.to(torch.bfloat16)
    ctx = torch.empty(B * rows, d_m, device="cuda", dtype=torch.bfloat16)
    scale = 0.5
    capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, scale,
                                                ctx.data_ptr(), kernel, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = decode_ref(qp, H, rows, scale)
    err = (ctx.float() - want).abs().max().item() / want.abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("kernel", [1, 0])
def test_decode_ragged_garbage_padding(kernel):
    import torch

    L, capi = _testing_lib()
    B, rows, n, d_m = 4, 64, 200, 1024
    g = torch.Generator(device="cuda").manual_seed(9)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    npi = torch.tensor([200, 1, 33, 150], dtype=torch.int32, device="cuda")
    Hg = H.clone()
    for b in range(B):
        Hg[b, int(npi[b]):] = float("nan")  # padding is garbage, even NaN
    ctx = torch.empty(B * rows, d_m, device="cuda", dtype=torch.bfloat16)
    capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), Hg.data_ptr(), npi.data_ptr(), B, rows, n, d_m,
                                                0.125, ctx.data_ptr(), kernel,
                                                torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = decode_ref(qp, H, rows, 0.125, npi)
    assert torch.isfinite(ctx.float()).all()
    err = (ctx.float() - want).abs().max().item() / want.abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("B,rows,n,d_m", [
    (1, 64, 1024, 1024),    # one input split over several clusters (stream-K, 4 segments)
    (20, 64, 1024, 1024),   # short last round -> stream-K chunks cut inputs
    (75, 64, 1024, 1024),   # 74 clusters + 1: stream-K
    (3, 64, 2000, 1024),    # long context: many segments per input (kMaxSegs guard)
    (2, 16, 130, 512),      # rows < 64 and a masked last tile in a split input
])
def test_decode_stream_k_schedules(B, rows, n, d_m):
    """The stream-K schedule (inputs split across clusters, partial records merged inside
    the decode kernel by the last segment to finish) against torch fp32, against the whole-input schedule (the same
    inputs passed with n_per_input), and run-to-run determinism."""
    import torch

    L, capi = _testing_lib()
    g = torch.Generator(device="cuda").manual_seed(B * 7 + n)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for npi in (None, None, torch.full((B,), n, dtype=torch.int32, device="cuda")):
        ctx = torch.full((B * rows, d_m), float("nan"), device="cuda", dtype=torch.bfloat16)
        capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(),
                                                    npi.data_ptr() if npi is not None else None, B, rows, n, d_m,
                                                    0.125, ctx.data_ptr(), 1, st))
        torch.cuda.synchronize()
        outs.append(ctx.float())
    want = decode_ref(qp, H, rows, 0.125)
    for o in outs:
        assert torch.isfinite(o).all()
        assert (o - want).abs().max().item() / want.abs().max().item() < 2e-2
    assert torch.equal(outs[0], outs[1])  # deterministic merge order
    assert (outs[0] - outs[2]).abs().max().item() / want.abs().max().item() < 1e-2


def test_decode_virtual_inputs_ragged():
    """rows > 64 (beam 12) with ragged n_per_input: every virtual input takes its real
    input's context length."""
    import torch

    L, capi = _testing_lib()
    B, rows, n, d_m = 3, 192, 200, 1024
    g = torch.Generator(device="cuda").manual_seed(13)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    npi = torch.tensor([200, 5, 97], dtype=torch.int32, device="cuda")
    Hg = H.clone()
    for b in range(B):
        Hg[b, int(npi[b]):] = float("nan")
    ctx = torch.empty(B * rows, d_m, device="cuda", dtype=torch.bfloat16)
    capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), Hg.data_ptr(), npi.data_ptr(), B, rows, n, d_m,
                                                0.125, ctx.data_ptr(), 1, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = decode_ref(qp, H, rows, 0.125, npi)
    assert torch.isfinite(ctx.float()).all()
    assert (ctx.float() - want).abs().max().item() / want.abs().max().item() < 2e-2


def test_decode_schedules_agree_over_random_batches():
    """Stream-K (short last round) and whole-input schedules agree for a sweep of batch
    sizes / context lengths around the 74-cluster boundaries (first-boundary-in-input and
    record-slot bookkeeping of the in-kernel merge), and the result matches torch fp32."""
    import torch

    L, capi = _testing_lib()
    rng = np.random.default_rng(5)
    cases = [(1, 1024), (7, 100), (37, 64), (73, 1024), (74, 300), (75, 1024), (111, 33), (148, 257),
             (150, 1024), (222, 96)] + [(int(b), int(n)) for b, n in zip(rng.integers(1, 200, 6),
                                                                       rng.choice([32, 130, 511, 1024], 6))]
    st = torch.cuda.current_stream().cuda_stream
    for B, n in cases:
        rows, d_m = 64, 512
        g = torch.Generator(device="cuda").manual_seed(B * 31 + n)
        qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
        H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        outs = []
        for npi in (None, torch.full((B,), n, dtype=torch.int32, device="cuda")):
            ctx = torch.full((B * rows, d_m), float("nan"), device="cuda", dtype=torch.bfloat16)
            capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(),
                                                        npi.data_ptr() if npi is not None else None, B, rows, n, d_m,
                                                        0.125, ctx.data_ptr(), 1, st))
            torch.cuda.synchronize()
            outs.append(ctx.float())
        assert torch.isfinite(outs[0]).all(), (B, n)
        scale = outs[1].abs().max().item()
        assert (outs[0] - outs[1]).abs().max().item() / scale < 1e-2, (B, n)
        sel = torch.tensor(sorted({0, B // 2, B - 1}), device="cuda")
        want = decode_ref(qp.view(B, rows, d_m)[sel].reshape(-1, d_m), H[sel], rows, 0.125)
        got = outs[0].view(B, rows, d_m)[sel].reshape(-1, d_m)
        assert (got - want).abs().max().item() / want.abs().max().item() < 2e-2, (B, n)


def test_decode_instrumented_instantiation_matches():
    """The instrumented decode instantiation (selected while the clock64 trace hook is set)
    computes bit-identical outputs to the production one, and records stamps."""
    import torch

    L, capi = _testing_lib()
    L.elattn_gpu_testing_set_decode_trace.argtypes = [ctypes.c_void_p]
    B, rows, n, d_m = 80, 64, 300, 1024  # stream-K / split schedule, masked last tile
    g = torch.Generator(device="cuda").manual_seed(21)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    tr = torch.zeros(2 * 32 * 64 + 4096, dtype=torch.int64, device="cuda")
    outs = []
    for trace in (None, tr):
        L.elattn_gpu_testing_set_decode_trace(trace.data_ptr() if trace is not None else None)
        ctx = torch.full((B * rows, d_m), float("nan"), device="cuda", dtype=torch.bfloat16)
        capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, 0.125,
                                                    ctx.data_ptr(), 1, st))
        torch.cuda.synchronize()
        outs.append(ctx)
    L.elattn_gpu_testing_set_decode_trace(None)
    assert torch.equal(outs[0], outs[1])
    assert int((tr != 0).sum()) > 0


@pytest.mark.parametrize("M,N,K,Z,split", [
    (128, 128, 64, 1, 0), (300, 1024, 1024, 1, 1),   # Q = Y.W_Q (fp32 path), M tail, split out
    (64, 1000, 1024, 4, 0),                          # scores q'.H^T per input (N tail)
    (64, 1024, 320, 3, 1),                           # C = P.H^T-copy per input, split out
    (77, 64, 4096, 2, 0),                            # long K: chunked accumulation keeps fp32 accuracy
])
def test_tf32x3_gemm_vs_fp64(M, N, K, Z, split):
    """The fp32 path's 3xTF32 tensor-core GEMM (split epilogue) against an fp64 reference:
    fp32-class accuracy independent of K (each 32-wide k-block is its own MMA chain)."""
    mn = 0
    import torch

    L, capi = _testing_lib()
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.elattn_gpu_testing_gemm_tf32x3.argtypes = [vp, i64, i64, vp, i64, i64, vp, vp, i64, i64, vp, i64,
                                                 i32, i32, i32, i32, ctypes.c_float, vp]
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.rand(Z, M, K, generator=g, device="cuda") * 2 - 1
    Bm = torch.rand(Z, K, N, generator=g, device="cuda") * 2 - 1 if mn else \
        torch.rand(Z, N, K, generator=g, device="cuda") * 2 - 1
    bias = torch.rand(Z, N, generator=g, device="cuda")
    C = torch.zeros(Z, M, N, device="cuda")
    C2 = torch.zeros_like(C) if split else None
    ldb, sBz = (N, K * N) if mn else (K, N * K)
    capi.check(L.elattn_gpu_testing_gemm_tf32x3(A.data_ptr(), K, M * K, Bm.data_ptr(), ldb, sBz, C.data_ptr(),
                                                C2.data_ptr() if split else None, N, M * N, bias.data_ptr(), N,
                                                M, N, K, Z, 0.75, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    Bk = Bm.double().transpose(1, 2) if mn else Bm.double()
    want = 0.75 * torch.einsum("zmk,znk->zmn", A.double(), Bk) + bias.double()[:, None, :]
    got = C.double() + (C2.double() if split else 0)
    err = ((got - want).abs().max() / want.abs().max()).item()
    assert err < 2e-6, err


@pytest.mark.parametrize("B", [20, 75, 320])
def test_decode_split_records_garbage_workspace_and_graph_replay(B):
    """Split inputs keep their partial records in the caller's workspace: a workspace full
    of garbage bytes, a reused one, and repeated replays of a captured step all give the
    bits of a fresh run.
    B = 20 / 75: stream-K; B = 320: tail-split (4 full rounds + 24 inputs in 3 parts)."""
    import torch

    import paper_2105_04779_b200 as E
    from paper_2105_04779_b200 import capi

    h, d_m, d_k, x, n = 16, 1024, 64, 4, 1024
    layer = E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(3)), E.DTYPE_BF16)
    g = torch.Generator(device="cuda").manual_seed(B)
    H = (torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Y = (torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    L = capi.lib()
    need = layer.dev.workspace_size(B, x, n)
    st = torch.cuda.current_stream()

    def run(ws, out):
        capi.check(L.elattn_gpu_el_attention_step(layer.dev.handle, Y.data_ptr(), H.data_ptr(), None, B, x, n,
                                                  out.data_ptr(), ws.data_ptr(), need, st.cuda_stream))

    ref = torch.empty_like(Y)
    run(torch.zeros(need, dtype=torch.uint8, device="cuda"), ref)
    for fill in (0xFF, 0x5A):
        ws = torch.full((need,), fill, dtype=torch.uint8, device="cuda")
        for _ in range(2):  # reused workspace: counters left reset by the previous launch
            out = torch.full_like(Y, float("nan"))
            run(ws, out)
            torch.cuda.synchronize()
            assert torch.equal(out, ref), fill
    ws = torch.randint(0, 256, (need,), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.full_like(Y, float("nan"))
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s2):
            capi.check(L.elattn_gpu_el_attention_step(layer.dev.handle, Y.data_ptr(), H.data_ptr(), None, B, x, n,
                                                      out.data_ptr(), ws.data_ptr(), need, s2.cuda_stream))
    for _ in range(3):
        out.fill_(float("nan"))
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


@pytest.mark.parametrize("B,rows,d_m", [(5, 64, 1024), (37, 64, 512), (150, 64, 512), (9, 192, 1024)])
def test_decode_ragged_schedules(B, rows, d_m):
    """Ragged batches under every schedule: longest-first whole inputs (the automatic
    choice: in-kernel counting sort by tile count, boustrophedon over the clusters), ragged
    stream-K (chunks of the inputs' own tiles, split inputs merged in cluster order) and
    strided whole inputs.  Against torch fp32 with NaN padding past n_b; deterministic."""
    import torch

    L, capi = _testing_lib()
    L.elattn_gpu_testing_decode_sched.argtypes = [ctypes.c_int]
    n = 700
    g = torch.Generator(device="cuda").manual_seed(B * 3 + rows)
    qp = (torch.randn(B * rows, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    npi = torch.randint(1, n + 1, (B,), generator=g, device="cuda", dtype=torch.int32)
    npi[0] = n
    Hg = H.clone()
    for b in range(B):
        Hg[b, int(npi[b]):] = float("nan")
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    try:
        for mode in (0, 0, 2, 1, 1):
            capi.check(L.elattn_gpu_testing_decode_sched(mode))
            ctx = torch.full((B * rows, d_m), float("nan"), device="cuda", dtype=torch.bfloat16)
            capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), Hg.data_ptr(), npi.data_ptr(), B, rows, n, d_m,
                                                        0.125, ctx.data_ptr(), 1, st))
            torch.cuda.synchronize()
            outs.append(ctx.float())
    finally:
        capi.check(L.elattn_gpu_testing_decode_sched(0))
    want = decode_ref(qp, H, rows, 0.125, npi)
    for o in outs:
        assert torch.isfinite(o).all()
        assert (o - want).abs().max().item() / want.abs().max().item() < 2e-2
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[3], outs[4])
    for o in outs[2:]:
        assert (outs[0] - o).abs().max().item() / want.abs().max().item() < 1e-2


@pytest.mark.parametrize("R,d_m,h", [(128, 1024, 16), (256, 1024, 16), (77, 1024, 16), (200, 512, 8), (4, 1024, 16)])
def test_fused_query_expansion(R, d_m, h):
    """The fused small-batch query expansion (one launch: every CTA computes the bf16 Q_i
    tile on the tensor cores, then its quarter of q' = Q_i.W_K,i^T) against torch fp32 of
    (bf16(Y.W_Q + b_Q))_i.W_K,i^T, against the two-GEMM path, and run-to-run identical."""
    import torch

    import paper_2105_04779_b200 as E
    from paper_2105_04779_b200 import capi

    L = capi.lib()
    L.elattn_gpu_testing_qexp_fused.argtypes = [ctypes.c_int]
    d_k = 64
    p = E.AttentionParams.random(h, d_m, d_k, E.Rng(R + d_m))
    layer = E.ElAttentionLayer(p, E.DTYPE_BF16)
    g = torch.Generator(device="cuda").manual_seed(R)
    Y = (torch.rand((R, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    outs = []
    try:
        for mode in (1, 1, 0):
            capi.check(L.elattn_gpu_testing_qexp_fused(mode))
            outs.append(layer.build_el_query(Y).float())
            torch.cuda.synchronize()
    finally:
        capi.check(L.elattn_gpu_testing_qexp_fused(-1))
    Wq = torch.from_numpy(np.asarray(p.Wq)).cuda().to(torch.bfloat16).float()   # [h][d_m][d_k]
    Wk = torch.from_numpy(np.asarray(p.Wk)).cuda().to(torch.bfloat16).float()
    bq = torch.from_numpy(np.asarray(p.bq)).cuda().float().view(h, d_k)
    Q = (torch.einsum("rd,hdk->rhk", Y.float(), Wq) + bq[None]).to(torch.bfloat16).float()
    want = torch.einsum("rhk,hdk->rhd", Q, Wk).reshape(R * h, d_m)
    scale = want.abs().max().item()
    for o in outs:
        assert (o - want).abs().max().item() / scale < 1e-2
    assert torch.equal(outs[0], outs[1])
    assert (outs[0] - outs[2]).abs().max().item() / scale < 1e-2
