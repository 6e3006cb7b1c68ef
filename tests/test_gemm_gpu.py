"""tcgen05/TMEM/TMA GEMMs (K1 router GEMM, K6 expert FFN) against a plain
PyTorch fp32 reference of the same op.

Tolerances: fp32 outputs of bf16 x bf16 products with fp32 accumulation —
|err| <= 1e-3 * max|ref| + 1e-3; bf16 outputs — max|err| / max|ref| <= 1e-2
(north-star bf16 tolerance)."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_16947_b200 import _lib

    return _lib


def _gemm(L, A, B, out_kind):
    M, K = A.shape
    N = B.shape[0]
    D = torch.empty(M, N, dtype=torch.float32 if out_kind == 0 else torch.bfloat16, device="cuda")
    L.check(L.lib().hep_gemm_bf16(A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, out_kind, L.stream_handle()), "gemm")
    torch.cuda.synchronize()
    return D


@pytest.mark.parametrize("M,N,K", [(128, 16, 64), (300, 16, 512), (1000, 32, 256), (257, 64, 128), (4096, 128, 2048),
                                   (777, 256, 1024), (4096, 256, 7168), (130, 48, 64)])
def test_dense_fp32_out(L, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
    D = _gemm(L, A, B, 0)
    ref = A.float() @ B.float().T
    err = (D - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1000, 512, 512), (4096, 1024, 4096)])
def test_dense_bf16_out(L, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
    D = _gemm(L, A, B, 1).float()
    ref = A.float() @ B.float().T
    assert (D - ref).abs().max().item() / ref.abs().max().item() <= 1e-2


def _ffn_ref(x, w1, w3, w2):
    h = torch.nn.functional.silu(x @ w1.T) * (x @ w3.T)
    return h.to(torch.bfloat16).float() @ w2.T


@pytest.mark.parametrize("E,d,F,sizes", [
    (4, 512, 1024, [300, 0, 129, 1000]),
    (3, 256, 384, [1, 128, 255]),
    (8, 1024, 768, [513, 64, 2000, 7, 0, 128, 300, 900]),
])
def test_grouped_expert_ffn(L, E, d, F, sizes):
    from paper_2511_16947_b200.layer import init_expert_weights, interleave_w13

    dev = "cuda"
    w1, w2, w3 = init_expert_weights(E, d, F, seed=3, device=dev)
    w13 = interleave_w13(w1, w3)
    # segments in an arbitrary expert order (two segments per expert, like two dst GPUs)
    segs, row = [], 0
    for rep in range(2):
        for e in reversed(range(E)):
            n = sizes[e] if rep == 0 else sizes[e] // 3
            segs.append((row, n, e, rep))
            row += n
    R = row
    x = torch.randn(max(R, 1), d, device=dev).to(torch.bfloat16)
    seg = torch.tensor(segs, dtype=torch.int32, device=dev)
    h = torch.empty(max(R, 1), F, dtype=torch.bfloat16, device=dev)
    y = torch.full((max(R, 1), d), float("nan"), dtype=torch.bfloat16, device=dev)
    lib = L.lib()
    ws = torch.empty(int(lib.hep_moe_ffn_workspace(len(segs), R, E)), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    L.check(lib.hep_moe_expert_ffn(x.data_ptr(), w13.data_ptr(), w2.data_ptr(), seg.data_ptr(), len(segs), R, d, F, E,
                                   h.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), st.data_ptr(),
                                   L.stream_handle()), "ffn")
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    for (r0, n, e, _) in segs:
        if n == 0:
            continue
        ref = _ffn_ref(x[r0:r0 + n].float(), w1[e].float(), w3[e].float(), w2[e].float())
        got = y[r0:r0 + n].float()
        assert torch.isfinite(got).all()
        rel = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
        assert rel <= 1e-2, (e, n, rel)


def _run_ffn(L, x, w13, w2, segs, R, d, F, E):
    dev = x.device
    seg = torch.tensor(segs, dtype=torch.int32, device=dev)
    h = torch.empty(max(R, 1), F, dtype=torch.bfloat16, device=dev)
    y = torch.full((max(R, 1), d), float("nan"), dtype=torch.bfloat16, device=dev)
    lib = L.lib()
    ws = torch.empty(int(lib.hep_moe_ffn_workspace(len(segs), R, E)), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    L.check(lib.hep_moe_expert_ffn(x.data_ptr(), w13.data_ptr(), w2.data_ptr(), seg.data_ptr(), len(segs), R, d, F, E,
                                   h.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), st.data_ptr(),
                                   L.stream_handle()), "ffn")
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    return h, y


@pytest.mark.parametrize("E,d,F", [(24, 512, 768), (40, 256, 256), (12, 512, 1024)])
def test_grouped_ffn_skewed_sizes_pair_and_single(L, E, d, F, tune):
    """Skewed expert sizes as a Zipf gate produces them: most experts carry a handful
    of rows (one partial m-tile), a few carry many tiles with a partial tail.  Both the
    1-CTA kernel (128-row tiles) and the CTA-pair kernel (256-row tiles) are checked
    against fp32 torch, and must agree bit for bit (each output element is the same
    K-ordered dot product whatever tile it lands in)."""
    from paper_2511_16947_b200.layer import init_expert_weights, interleave_w13

    dev = "cuda"
    w1, w2, w3 = init_expert_weights(E, d, F, seed=5, device=dev)
    w13 = interleave_w13(w1, w3)
    base = [0, 1, 2, 15, 16, 17, 31, 33, 64, 65, 100, 111, 112, 113, 127, 128, 129, 255, 257, 320, 700, 1500]
    sizes = [base[(7 * e) % len(base)] for e in range(E)]
    segs, row = [], 0
    for e in reversed(range(E)):  # one contiguous segment per expert, arbitrary expert order
        segs.append((row, sizes[e], e, 0))
        row += sizes[e]
    R = row
    x = torch.randn(R, d, device=dev).to(torch.bfloat16)
    outs = {}
    for pair in ("0", "1"):
        tune(ffn_pair=int(pair))
        outs[pair] = _run_ffn(L, x, w13, w2, segs, R, d, F, E)
    for pair in ("0", "1"):
        h, y = outs[pair]
        for (r0, n, e, _) in segs:
            if n == 0:
                continue
            ref = _ffn_ref(x[r0:r0 + n].float(), w1[e].float(), w3[e].float(), w2[e].float())
            got = y[r0:r0 + n].float()
            assert torch.isfinite(got).all()
            rel = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
            assert rel <= 1e-2, (pair, e, n, rel)
    assert torch.equal(outs["0"][0], outs["1"][0])
    assert torch.equal(outs["0"][1], outs["1"][1])


def test_grouped_ffn_light_expert_split(L, tune):
    """CTA pairs with the light experts (<= hep_tuning.ffn_light_rows rows) split off to the
    1-CTA kernel on their own tile list: every threshold (none, 128, 256, all experts
    light) gives the same bytes, and hep_moe_ffn_launches reports the extra launches."""
    from paper_2511_16947_b200.layer import init_expert_weights, interleave_w13

    E, d, F = 48, 256, 512
    w1, w2, w3 = init_expert_weights(E, d, F, seed=7, device="cuda")
    w13 = interleave_w13(w1, w3)
    base = [0, 3, 64, 127, 128, 129, 200, 256, 257, 700, 1500, 2100]
    sizes = [base[(5 * e) % len(base)] for e in range(E)]
    segs, row = [], 0
    for e in range(E):  # two segments per expert (two source GPUs), contiguous rows
        a = sizes[e] // 3
        segs += [(row, a, e, 0), (row + a, sizes[e] - a, e, 1)]
        row += sizes[e]
    R = row
    x = torch.randn(R, d, device="cuda").to(torch.bfloat16)
    tune(ffn_pair=1)
    outs = {}
    for lr in ("0", "128", "256", "100000"):
        tune(ffn_light_rows=int(lr))
        outs[lr] = _run_ffn(L, x, w13, w2, segs, R, d, F, E)
        assert int(L.lib().hep_moe_ffn_launches(R, E, 0)) == (4 if lr == "0" else 8)
    for lr in ("128", "256", "100000"):
        assert torch.equal(outs[lr][0], outs["0"][0]) and torch.equal(outs[lr][1], outs["0"][1]), lr
    r0, n = segs[2 * 9][0], sizes[9]  # spot-check one heavy expert against fp32 torch
    ref = _ffn_ref(x[r0:r0 + n].float(), w1[9].float(), w3[9].float(), w2[9].float())
    assert (outs["128"][1][r0:r0 + n].float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("T,d,E,K,G,bias", [
    (4096, 512, 8, 2, 4, True), (2000, 256, 8, 1, 2, False), (4096, 1024, 40, 6, 8, True),
    (8192, 512, 128, 8, 8, True), (3000, 512, 128, 8, 3, False), (4096, 768, 200, 8, 8, True),
    (2048, 512, 256, 8, 8, True), (1024, 256, 512, 8, 4, True), (1024, 256, 64, 10, 4, True),
    (2048, 256, 20, 3, 10, True), (1024, 512, 48, 5, 2, False), (1024, 256, 32, 7, 4, True),
    (16384, 512, 8, 2, 8, True), (32768, 256, 128, 8, 8, True), (16384, 256, 256, 8, 8, True),
])
@pytest.mark.parametrize("tile,mc,pair", [(0, 0, 0), (0, 1, 1), (0, 2, 1), (0, 4, 1), (128, 1, 1), (80, 4, 0),
                                          (48, 2, 0), (0, 0, 2)])
def test_router_topk_fused_equals_unfused(L, T, d, E, K, G, bias, tile, mc, pair, tune):
    """hep_router_topk (gate in the router GEMM's epilogue) against the unfused chain
    hep_gemm_bf16 -> hep_gate_topk -> hep_gate_chunk_counts: logits, top-K indices,
    weights, histogram and per-64-token chunk counts bit for bit (E > 256 and K > 8 take
    the unfused path inside the same entry point).  tile = router rows per CTA tile
    (0 = the automatic all-SM split, e.g. 112 rows at 16384 tokens; 80 / 48: tiles that
    cut through 64-token chunks, whose counts then go through global atomics); the gate
    epilogue runs on both column halves (merged through shared memory) when E_pad % 32 == 0.
    mc = hep_tuning.router_mc: clusters of mc CTAs sharing each Wg tile by TMA multicast
    (0 = auto; tile counts that are not a multiple of mc leave empty tiles in the last
    cluster).  pair = hep_tuning.router_pair: 0 auto / 2 on = CTA pairs (256 tokens per
    pair, half the Wg tile per CTA) for E_pad > 64, 1 = the 1-CTA kernel."""
    tune(router_tile_rows=tile, router_mc=mc, router_pair=pair)
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(T + E + K)
    e_pad = max(16, (E + 15) // 16 * 16)
    e64 = (E + 63) // 64 * 64
    x = torch.randn(T, d, generator=g, device=dev).to(torch.bfloat16)
    wg = torch.zeros(max(e64, e_pad), d, dtype=torch.bfloat16, device=dev)
    wg[:E] = (torch.randn(E, d, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    # duplicate two experts' rows so exact ties occur (ties -> lower expert id)
    wg[E - 1] = wg[0]
    b = (torch.randn(E, generator=g, device=dev) * 0.5).float() if bias else None
    if b is not None:
        b[E - 1] = b[0]
    tps = (T + G - 1) // G
    ncs = (tps + 63) // 64
    lib = L.lib()
    s = L.stream_handle()

    def bufs():
        return (torch.full((T, e_pad), float("nan"), device=dev), torch.full((T, K), -1, dtype=torch.int32, device=dev),
                torch.full((T, K), float("nan"), device=dev), torch.zeros(G, E, dtype=torch.int64, device=dev),
                torch.full((G * ncs * E,), -7, dtype=torch.int32, device=dev))

    lg0, i0, w0, h0, c0 = bufs()
    L.check(lib.hep_gemm_bf16(x.data_ptr(), wg.data_ptr(), lg0.data_ptr(), T, e_pad, d, 0, s), "gemm")
    L.check(lib.hep_gate_topk(lg0.data_ptr(), e_pad, L.ptr(b), T, E, K, tps, G, i0.data_ptr(), w0.data_ptr(),
                              h0.data_ptr(), s), "gate")
    L.check(lib.hep_gate_chunk_counts(i0.data_ptr(), T, K, E, tps, G, c0.data_ptr(), s), "chunks")
    lg1, i1, w1, h1, c1 = bufs()
    L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, L.ptr(b), K, tps, G, lg1.data_ptr(),
                                i1.data_ptr(), w1.data_ptr(), h1.data_ptr(), c1.data_ptr(), s), "router_topk")
    torch.cuda.synchronize()
    assert torch.equal(lg0, lg1)
    assert torch.equal(i0, i1)
    assert torch.equal(w0, w1)
    assert torch.equal(h0, h1)
    assert int(h1.sum()) == T * K
    assert torch.equal(c0, c1)
    # and without the logits buffer (fused path only)
    if E <= 256 and K <= 8:
        _, i2, w2, h2, c2 = bufs()
        L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, L.ptr(b), K, tps, G, None,
                                    i2.data_ptr(), w2.data_ptr(), h2.data_ptr(), c2.data_ptr(), s), "router_topk")
        torch.cuda.synchronize()
        assert torch.equal(i0, i2) and torch.equal(w0, w2) and torch.equal(h0, h2) and torch.equal(c0, c2)


@pytest.mark.parametrize("T,d,E,K,G,pair", [(4096, 512, 8, 2, 4, 0), (8192, 512, 128, 8, 8, 0),
                                            (4096, 768, 256, 8, 8, 0), (4096, 768, 256, 8, 8, 1), (3000, 256, 40, 6, 3, 0)])
def test_router_topk_ws_zeroes_in_kernel(L, T, d, E, K, G, pair, tune):
    """hep_router_topk_ws (the kernel's CTA 0 zeroes the histogram, the others add after it,
    self-resetting sync words) equals hep_router_topk (separate zeroing launch) on a histogram
    buffer full of garbage, leaves the sync words zero, and replays inside a CUDA graph."""
    tune(router_pair=pair)
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(T + E)
    e_pad = max(16, (E + 15) // 16 * 16)
    x = torch.randn(T, d, generator=g, device=dev).to(torch.bfloat16)
    wg = torch.zeros(max(64, e_pad), d, dtype=torch.bfloat16, device=dev)
    wg[:E] = (torch.randn(E, d, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    tps = (T + G - 1) // G
    lib, s = L.lib(), L.stream_handle()
    assert int(lib.hep_router_sync_bytes()) <= 16

    def run(ws, h, sync=None, stream=s):
        lg = torch.empty(T, e_pad, device=dev)
        i = torch.empty(T, K, dtype=torch.int32, device=dev)
        w = torch.empty(T, K, device=dev)
        if ws:
            L.check(lib.hep_router_topk_ws(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, None, K, tps, G, lg.data_ptr(),
                                           i.data_ptr(), w.data_ptr(), h.data_ptr(), None, sync.data_ptr(), stream), "ws")
        else:
            L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, None, K, tps, G, lg.data_ptr(),
                                        i.data_ptr(), w.data_ptr(), h.data_ptr(), None, stream), "router")
        return i, w

    h0 = torch.full((G, E), 12345, dtype=torch.int64, device=dev)
    i0, w0 = run(False, h0)
    sync = torch.zeros(4, dtype=torch.int32, device=dev)
    for _ in range(3):
        h1 = torch.full((G, E), -777, dtype=torch.int64, device=dev)
        i1, w1 = run(True, h1, sync)
        torch.cuda.synchronize()
        assert torch.equal(h0, h1) and torch.equal(i0, i1) and torch.equal(w0, w1)
        assert int(sync.abs().sum()) == 0
    h2 = torch.full((G, E), 99, dtype=torch.int64, device=dev)
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        gr.capture_begin()
        run(True, h2, sync, stream=cs.cuda_stream)
        gr.capture_end()
    for _ in range(3):
        h2.fill_(-5)
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(h0, h2)
        assert int(sync.abs().sum()) == 0


@pytest.mark.parametrize("T,d,E,K,G", [(16384, 4096, 8, 2, 8), (32768, 2048, 128, 8, 8), (16384, 7168, 256, 8, 8)])
def test_router_topk_ws_fullsize_equals_unfused(L, T, d, E, K, G):
    """The BASELINE shapes (Mixtral / Qwen3 / DeepSeek-V3) with the default launch tuning
    (DeepSeek-V3 on the CTA-pair router kernel) through hep_router_topk_ws, the entry point
    the layer uses, against the unfused chain: logits, top-K, weights, histogram and chunk
    counts bit for bit, with a Zipf-skewed selection bias as in the bench."""
    import paper_2511_16947_b200 as P

    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(T + E)
    e_pad = max(16, (E + 15) // 16 * 16)
    x = torch.randn(T, d, generator=g, device=dev).to(torch.bfloat16)
    wg = torch.zeros(max(64, e_pad), d, dtype=torch.bfloat16, device=dev)
    wg[:E] = (torch.randn(E, d, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    b = torch.tensor(P.zipf_gate_bias(E, 1.0, 0), dtype=torch.float32, device=dev)
    tps = T // G
    ncs = tps // 64
    lib, s = L.lib(), L.stream_handle()

    def bufs():
        return (torch.full((T, e_pad), float("nan"), device=dev), torch.full((T, K), -1, dtype=torch.int32, device=dev),
                torch.full((T, K), float("nan"), device=dev), torch.full((G, E), 77, dtype=torch.int64, device=dev),
                torch.full((G * ncs * E,), -7, dtype=torch.int32, device=dev))

    lg0, i0, w0, h0, c0 = bufs()
    h0.zero_()
    L.check(lib.hep_gemm_bf16(x.data_ptr(), wg.data_ptr(), lg0.data_ptr(), T, e_pad, d, 0, s), "gemm")
    L.check(lib.hep_gate_topk(lg0.data_ptr(), e_pad, b.data_ptr(), T, E, K, tps, G, i0.data_ptr(), w0.data_ptr(),
                              h0.data_ptr(), s), "gate")
    L.check(lib.hep_gate_chunk_counts(i0.data_ptr(), T, K, E, tps, G, c0.data_ptr(), s), "chunks")
    lg1, i1, w1, h1, c1 = bufs()
    sync = torch.zeros(4, dtype=torch.int32, device=dev)
    L.check(lib.hep_router_topk_ws(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G, lg1.data_ptr(),
                                   i1.data_ptr(), w1.data_ptr(), h1.data_ptr(), c1.data_ptr(), sync.data_ptr(), s), "ws")
    torch.cuda.synchronize()
    assert torch.equal(lg0, lg1) and torch.equal(i0, i1) and torch.equal(w0, w1)
    assert torch.equal(h0, h1) and int(h1.sum()) == T * K
    assert torch.equal(c0, c1)
    assert int(sync.abs().sum()) == 0
