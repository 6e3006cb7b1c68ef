"""BASELINE configs[4] (scheduler + dispatch stress: Zipf skew 0-2, tokens 4K-1M, G = 2/4/8)
at its corners, through the whole layer on the B200.

At 1M tokens the oracle's per-token assignment loop (`oracle/layer_ref.py:45-82`) is too
slow, so the checks are the size-independent ones:
  * routing decisions (top-K of the device's logits + the Zipf bias) and the per-source
    histogram: bit-exact against `layer_ref.topk_select` / `histogram` (numpy, vectorised);
  * the schedule (m, integerized plan, Algorithm-1 ranges, per-GPU loads): bit-exact
    against the C Dinic oracle on that histogram;
  * the token -> receive-row map: a bijection onto the receive rows; every token's row in
    its expert's block; the (expert, source, destination) token counts it realises equal
    the routing table's; row_tok is its inverse;
  * the permute: bit-exact copies (rows[r] == x[row_tok[r]]);
  * the layer output on 64 sampled tokens against the fp32 SwiGLU restatement (bf16
    tolerance 1e-2, `layer_ref.expert_ffn`).
The exact per-token map is pinned against the oracle at small T in test_layer_gpu.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_16947_b200 as pkg

    return pkg


@pytest.mark.parametrize("G,E,K,T,s", [
    (8, 8, 2, 1 << 20, 2.0),      # Mixtral routing, 1M tokens, heaviest skew
    (8, 128, 8, 1 << 20, 0.0),    # Qwen3 routing, 1M tokens, uniform
    (2, 128, 8, 1 << 20, 2.0),    # 2 GPUs, 1M tokens, heaviest skew
    (4, 256, 8, 4096, 1.0),       # DeepSeek-V3 routing, smallest micro-batch
    (8, 256, 8, 262144, 1.5),
])
def test_stress_corner(P, oracle_lib, G, E, K, T, s):
    from oracle import layer_ref

    d, F = 256, 128
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
    layer = P.MoELayer(pl, d, F, K, seed=3, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(77), device="cuda").to(torch.bfloat16)
    out = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    b = layer.buffers(T)
    tps = T // G

    # routing + histogram: bit-exact
    logits = b.logits[:, :E].cpu().numpy()
    idx_ref, w_ref = layer_ref.topk_select(logits, K, None if bias is None else bias.numpy())
    idx = b.topk_idx.cpu().numpy()
    assert np.array_equal(idx, idx_ref)
    assert np.allclose(b.topk_w.cpu().numpy(), w_ref, rtol=1e-5, atol=1e-6)
    hist = layer_ref.histogram(idx_ref, E, G, tps)
    assert np.array_equal(b.hist.cpu().numpy(), hist)

    # schedule: bit-exact against the Dinic oracle on the same load matrix
    groups = [tuple(g) for g in pl.edp_groups]
    ref = oracle_lib.full_path(G, groups, hist.T.tolist(), None)
    sd = layer.sched
    assert sd.m[:2].cpu().tolist() == list(ref["m"])
    assert sd.rows(sd.xi) == ref["xi"]
    ranges = [tuple(r) for r in sd.host_ranges()]
    assert [list(r) for r in ranges] == [list(r) for r in ref["ranges"]]
    assert sd.gpu_load.cpu().tolist() == list(ref["gpu_load"])
    assert int(sd.m[3].item()) == ref["obj_int"] == max(ref["gpu_load"])  # integerized objective

    # token -> row map
    R = T * K
    tok_row = b.tok_row.cpu().numpy().astype(np.int64)
    assert np.array_equal(np.sort(tok_row.reshape(-1)), np.arange(R))
    row_tok = b.row_tok[:R].cpu().numpy()
    assert np.array_equal(row_tok[tok_row], np.repeat(np.arange(T)[:, None], K, axis=1))
    er = b.expert_rows.cpu().numpy()
    assert er[E] == R
    assert np.all((tok_row >= er[idx]) & (tok_row < er[idx + 1]))
    seg = b.seg[: b.n_seg].cpu().numpy().astype(np.int64)  # (row start, count, expert, gpu)
    p = np.searchsorted(seg[:, 0], tok_row.reshape(-1), side="right") - 1
    assert np.all(tok_row.reshape(-1) < seg[p, 0] + seg[p, 1])
    assert np.array_equal(seg[p, 2], idx.reshape(-1))
    got = np.zeros((E, G, G), dtype=np.int64)
    src = np.repeat(np.arange(T) // tps, K)
    np.add.at(got, (idx.reshape(-1), src, seg[p, 3]), 1)
    want = np.zeros((E, G, G), dtype=np.int64)
    for e, sr, dst, c in ranges:
        want[e, sr, dst] += c
    assert np.array_equal(got, want)

    # permute: exact copies
    assert torch.equal(b.rows[:R], x[b.row_tok[:R].long()])

    # output on sampled tokens (fp32 SwiGLU restatement, bf16 tolerance)
    rng = np.random.default_rng(T + E)
    toks = np.sort(rng.choice(T, size=64, replace=False))
    xs = x[torch.as_tensor(toks, device="cuda")].float().cpu().numpy()
    w1, w2, w3 = (w.float().cpu().numpy() for w in (layer.w1, layer.w2, layer.w3))
    want_out = np.zeros((len(toks), d), dtype=np.float32)
    for i, t in enumerate(toks):
        for k in range(K):
            e = idx_ref[t, k]
            y = layer_ref.expert_ffn(xs[i:i + 1], w1[e], w3[e], w2[e])
            want_out[i] += w_ref[t, k] * layer_ref.bf16_round(y)[0]
    have = out[torch.as_tensor(toks, device="cuda")].float().cpu().numpy()
    rel = np.abs(have - want_out).max() / np.abs(want_out).max()
    assert rel <= 1e-2, rel
