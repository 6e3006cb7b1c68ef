"""End-to-end MoE layer parity on the B200 against the CPU oracle.

Bit-exact: top-K routing decisions (on the device's own fp32 logits), the
per-(source, expert) histogram = load matrix, the whole schedule (m, plan,
integerized per-GPU loads, routing table) and the token -> receive-row
assignment.  Tolerance: router logits |err| <= 1e-3·max|ref| (fp32 accumulate
order), top-K weights 1e-5, layer output max|err|/max|ref| <= 1e-2 (bf16).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_16947_b200 as P

    return P


def _run(P, G, E, K, d, F, T, s=1.0, seed=0, sample=None, fuse_permute=False):
    from oracle import layer_ref

    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape) if E >= G else P.identical_placement(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, s, seed)) if s > 0 else None
    layer = P.MoELayer(pl, d, F, K, seed=seed, gate_bias=bias, fuse_permute=fuse_permute)
    g = torch.Generator(device="cuda").manual_seed(1000 + seed)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    out = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    b = layer.buffers(T)
    logits = b.logits[:, :E].cpu().numpy()
    ref = layer_ref.layer_forward(
        x.float().cpu().numpy(), logits, K, [tuple(gr) for gr in pl.edp_groups], G,
        layer.w1.float().cpu().numpy(), layer.w2.float().cpu().numpy(), layer.w3.float().cpu().numpy(),
        bias=None if bias is None else bias.numpy(), sample=sample,
    )
    return layer, x, out, b, ref, pl


def test_tiny_config_bit_exact_schedule_and_output(P):
    """BASELINE configs[0]: 8 experts top-2, d=512, ffn=1024, 4096 tokens,
    simulated EP=4, Zipf-skewed routing."""
    from oracle import layer_ref

    layer, x, out, b, ref, pl = _run(P, G=4, E=8, K=2, d=512, F=1024, T=4096, s=1.0)
    # router GEMM vs fp32
    lref = x.float() @ layer.wg[: layer.E].float().T
    lerr = (b.logits[:, : layer.E] - lref).abs().max().item()
    assert lerr <= 1e-3 * lref.abs().max().item() + 1e-4
    # routing decisions and loads: bit-exact
    assert np.array_equal(b.topk_idx.cpu().numpy(), ref["topk_idx"])
    assert np.allclose(b.topk_w.cpu().numpy(), ref["topk_w"], rtol=1e-5, atol=1e-6)
    assert np.array_equal(b.hist.cpu().numpy(), ref["hist"])
    sd = layer.sched
    assert sd.m[:2].cpu().tolist() == list(ref["sched"]["m"])
    assert sd.rows(sd.xi) == ref["sched"]["xi"]
    assert [list(r) for r in sd.host_ranges()] == [list(r) for r in ref["sched"]["ranges"]]
    assert sd.gpu_load.cpu().tolist() == ref["sched"]["gpu_load"]
    # token -> row schedule: bit-exact
    assert np.array_equal(b.tok_row.cpu().numpy(), ref["tok_row"])
    assert b.expert_rows.cpu().tolist() == ref["expert_rows"].tolist()
    # the permute writes exact copies, and the layer with the permute fused into the first
    # GEMM's TMA gather (hep_moe_expert_ffn_gather) gives the same output bit for bit
    R = x.shape[0] * layer.K
    assert torch.equal(b.rows[:R], x[b.row_tok[:R].long()])
    out2 = _run(P, G=4, E=8, K=2, d=512, F=1024, T=4096, s=1.0, fuse_permute=True)[2]
    assert torch.equal(out, out2)
    # layer output (bf16 tolerance)
    got = out.float().cpu().numpy()
    rel = np.abs(got - ref["out"]).max() / np.abs(ref["out"]).max()
    assert rel <= 1e-2, rel


@pytest.mark.parametrize("G,E,K,d,F,T,s", [
    (8, 8, 2, 1024, 512, 8192, 1.5),     # Mixtral-like routing, small dims
    (8, 128, 8, 512, 256, 8192, 1.0),    # Qwen3-like routing
    (8, 256, 8, 512, 256, 4096, 1.5),    # DeepSeek-like routing
    (2, 8, 2, 256, 128, 2048, 0.0),
])
def test_routing_shapes_sampled_output(P, G, E, K, d, F, T, s):
    rng = np.random.default_rng(G * E + T)
    sample = np.sort(rng.choice(T, size=96, replace=False))
    layer, x, out, b, ref, pl = _run(P, G, E, K, d, F, T, s=s, seed=1, sample=sample)
    fused = _run(P, G, E, K, d, F, T, s=s, seed=1, sample=sample[:4], fuse_permute=True)[2]
    assert torch.equal(out, fused)  # fused permute (TMA gather) == permute kernel + GEMM
    assert np.array_equal(b.topk_idx.cpu().numpy(), ref["topk_idx"])
    assert np.array_equal(b.hist.cpu().numpy(), ref["hist"])
    assert layer.sched.rows(layer.sched.xi) == ref["sched"]["xi"]
    assert np.array_equal(b.tok_row.cpu().numpy(), ref["tok_row"])
    got = out.float().cpu().numpy()[sample]
    rel = np.abs(got - ref["out"]).max() / np.abs(ref["out"]).max()
    assert rel <= 1e-2, rel


def test_repeatable_and_row_map_is_permutation(P):
    layer, x, out, b, ref, pl = _run(P, G=8, E=16, K=2, d=256, F=256, T=4096, s=0.5, seed=2)
    R = 4096 * 2
    rows = b.tok_row.flatten().cpu().numpy()
    assert np.array_equal(np.sort(rows), np.arange(R))
    out2 = layer(x).clone()
    assert torch.equal(out, out2)  # deterministic: no float atomics anywhere


def test_cuda_graph_replay_matches_eager(P):
    """The whole forward has no host sync: capture it once, refill the input in
    place with a differently routed batch, replay, and compare with eager."""
    layer, x, out, b, ref, pl = _run(P, G=8, E=16, K=2, d=256, F=256, T=4096, s=0.5, seed=3)
    graph = layer.capture(x)
    x2 = torch.randn(x.shape, generator=torch.Generator(device="cuda").manual_seed(99), device="cuda")
    x.copy_(x2.to(torch.bfloat16))
    graph.replay()
    torch.cuda.synchronize()
    got = b.out.clone()
    got_rows = b.tok_row.clone()
    eager = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    assert torch.equal(got_rows, b.tok_row)
    assert torch.equal(got, eager)
    assert not torch.equal(got, out)


@pytest.mark.parametrize("cfg", ["mixtral", "qwen3", "dsv3"])
def test_baseline_shapes_full_size(P, cfg):
    """BASELINE configs[1..3] at full size (EP=8 simulated on one device):
    routing, histogram, schedule and token->row map bit-exact against the CPU
    oracle; expert FFN + combine for 48 sampled tokens against a plain PyTorch
    fp32 reference of the same op (max|err|/max|ref| <= 1e-2)."""
    import bench
    from oracle import layer_ref

    E, K, d, F, T, G = bench.CONFIGS[cfg]
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(7), device="cuda").to(torch.bfloat16)
    out = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    b = layer.buffers(T)
    logits = b.logits[:, :E].cpu().numpy()
    idx, w = layer_ref.topk_select(logits, K, bias.numpy())
    assert np.array_equal(b.topk_idx.cpu().numpy(), idx)
    hist = layer_ref.histogram(idx, E, G, T // G)
    assert np.array_equal(b.hist.cpu().numpy(), hist)
    from oracle import oracle as O

    ref = O.full_path(G, pl.edp_groups, hist.T.copy())
    sd = layer.sched
    assert sd.m[:2].cpu().tolist() == list(ref["m"])
    assert sd.rows(sd.xq) == ref["xq"]
    assert sd.rows(sd.xi) == ref["xi"]
    assert [tuple(r) for r in sd.host_ranges()] == [tuple(r) for r in ref["ranges"]]
    tok_row, _ = layer_ref.receive_rows(pl.edp_groups, G, ref["xi"], ref["ranges"], idx, T // G)
    assert np.array_equal(b.tok_row.cpu().numpy(), tok_row)
    # sampled numerics, torch fp32 reference on the device
    rng = np.random.default_rng(3)
    toks = torch.tensor(np.sort(rng.choice(T, 48, replace=False)), device="cuda")
    xs = x[toks].float()
    ref_out = torch.zeros(len(toks), d, device="cuda")
    ti = b.topk_idx[toks].long()
    tw = b.topk_w[toks]
    for k in range(K):
        for e in ti[:, k].unique().tolist():
            sel = (ti[:, k] == e).nonzero().flatten()
            h = torch.nn.functional.silu(xs[sel] @ layer.w1[e].float().T) * (xs[sel] @ layer.w3[e].float().T)
            y = h.to(torch.bfloat16).float() @ layer.w2[e].float().T
            ref_out[sel] += tw[sel, k, None] * y.to(torch.bfloat16).float()
    got = out[toks].float()
    rel = ((got - ref_out).abs().max() / ref_out.abs().max()).item()
    assert rel <= 1e-2, rel
    del layer
    torch.cuda.empty_cache()


@pytest.mark.parametrize("ratio,kind", [(0.5, "cayley"), (0.3, "cayley"), (0.8, "identical"), (1.0, "cayley")])
def test_pipelined_split_layer(P, ratio, kind):
    """harmony_pipelined on the device: static share split evenly over replicas and
    assigned first (on a side stream, overlapping the scheduled phase's solve),
    scheduled share solved with gpu_base.  Both phases' schedules and the
    [expert][phase][dst][src][rank] token->row map bit-exact against the oracle; the
    layer output bit-identical to the single-phase layer (rows are independent in the
    GEMMs, combine sums k in a fixed order), eager and CUDA-graph replayed."""
    from fractions import Fraction

    from oracle import layer_ref
    from oracle import oracle as O

    G, E, K, d, F, T = 8, 16, 2, 256, 256, 4096
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape) if kind == "cayley" else P.identical_placement(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, 1.2, 1))
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(8), device="cuda").to(torch.bfloat16)
    plain = P.MoELayer(pl, d, F, K, seed=5, gate_bias=bias)
    ref_out = plain(x).clone()
    pip = P.MoELayer(pl, d, F, K, seed=5, gate_bias=bias, pipeline_ratio=ratio)
    out = pip(x).clone()
    torch.cuda.synchronize()
    pip.check_status()
    assert torch.equal(out, ref_out)
    b = pip.buffers(T)
    share = Fraction(1) - Fraction(ratio)
    loads = b.hist.cpu().numpy().T.tolist()
    f, lat = O.pipelined_path(G, [tuple(g) for g in pl.edp_groups], loads, share.numerator, share.denominator)
    ds = pip.sched
    assert ds.former.rows(ds.former.xi) == f["xi"]
    assert [tuple(r) for r in ds.former.host_ranges()] == [tuple(r) for r in f["ranges"]]
    assert ds.m[:2].cpu().tolist() == list(lat["m"])
    assert ds.rows(ds.xi) == lat["xi"]
    assert [tuple(r) for r in ds.host_ranges()] == [tuple(r) for r in lat["ranges"]]
    tok_row, n_rows = layer_ref.receive_rows_pipelined(pl.edp_groups, G, f, lat, f["loads"],
                                                       b.topk_idx.cpu().numpy(), T // G)
    assert n_rows == T * K
    assert np.array_equal(b.tok_row.cpu().numpy(), tok_row)
    # each phase's own row map: its rows, -1 for the other phase's assignments
    for ph in range(2):
        m = b.tok_row_ph[ph].cpu().numpy()
        own = m >= 0
        assert np.array_equal(m[own], tok_row[own])
    assert np.array_equal(b.tok_row_ph[0].cpu().numpy() >= 0, ~(b.tok_row_ph[1].cpu().numpy() >= 0))
    # the two-stream step captured as one CUDA graph, replayed on another micro-batch
    x2 = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(9), device="cuda").to(torch.bfloat16)
    ref2 = plain(x2).clone()
    xin = x.clone()
    g = pip.capture(xin)
    xin.copy_(x2)
    g.replay()
    torch.cuda.synchronize()
    pip.check_status()
    assert torch.equal(pip.buffers(T).out, ref2)


@pytest.mark.parametrize("G,E,K,d,F,T,case", [
    (8, 1024, 16, 256, 128, 2048, "max_experts_topk"),  # E and K at the ABI limits (unfused gate path)
    (10, 20, 3, 256, 128, 1000, "max_gpus_ragged"),     # G = HEP_MAX_GPUS, T not a multiple of 64/128
    (4, 8, 2, 256, 128, 4, "one_token_per_source"),
    (8, 64, 4, 256, 128, 2048, "all_tokens_to_k_experts"),  # every other expert empty
])
def test_edge_cases_against_oracle(P, G, E, K, d, F, T, case):
    """Edge cases of the path, whole layer against the oracle: routing, histogram,
    schedule and token->row map bit-exact, outputs within the bf16 tolerance."""
    from oracle import layer_ref

    shape = P.ClusterShape(G, E, 2)
    pl = (P.cayley_symmetric(shape) if (E & (E - 1)) == 0 and (G & (G - 1)) == 0
          else P.placement.symmetric_placement(shape))
    if case == "all_tokens_to_k_experts":
        bias = torch.full((E,), -30.0)
        bias[3:3 + K] = 30.0
    else:
        bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    layer = P.MoELayer(pl, d, F, K, seed=4, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(21), device="cuda").to(torch.bfloat16)
    out = layer(x).float().cpu().numpy()
    torch.cuda.synchronize()
    layer.check_status()
    b = layer.buffers(T)
    ref = layer_ref.layer_forward(
        x.float().cpu().numpy(), b.logits[:, :E].cpu().numpy(), K, [tuple(g) for g in pl.edp_groups], G,
        layer.w1.float().cpu().numpy(), layer.w2.float().cpu().numpy(), layer.w3.float().cpu().numpy(),
        bias=bias.numpy())
    assert np.array_equal(b.topk_idx.cpu().numpy(), ref["topk_idx"])
    assert np.array_equal(b.hist.cpu().numpy(), ref["hist"])
    assert layer.sched.rows(layer.sched.xi) == ref["sched"]["xi"]
    assert np.array_equal(b.tok_row.cpu().numpy(), ref["tok_row"])
    if case == "all_tokens_to_k_experts":
        assert int((b.hist.sum(dim=0) > 0).sum()) == K
    rel = np.abs(out - ref["out"]).max() / np.abs(ref["out"]).max()
    assert rel <= 1e-2, rel


def test_assignment_is_repeatable(P):
    """hep_moe_assign_precounted leaves the router's chunk counts intact: re-running the
    assignment on the same micro-batch reproduces the token->row map (regression: the
    chunk scan used to overwrite the counts in place)."""
    import ctypes

    from paper_2511_16947_b200 import _lib

    layer, x, out, b, ref, pl = _run(P, G=8, E=16, K=2, d=256, F=256, T=4096, s=0.5, seed=4)
    first = b.tok_row.clone()
    L = _lib.lib()
    for _ in range(3):
        _lib.check(L.hep_moe_assign_precounted(layer.sched.handle, ctypes.byref(layer.sched.out),
                                               b.topk_idx.data_ptr(), 4096, 2, 4096 // 8, b.row_align,
                                               b.tok_row.data_ptr(), b.row_tok.data_ptr(), b.seg.data_ptr(),
                                               b.expert_rows.data_ptr(), b.assign_ws.data_ptr(), b.assign_ws.numel(),
                                               _lib.stream_handle()), "assign")
    torch.cuda.synchronize()
    assert torch.equal(b.tok_row, first)
