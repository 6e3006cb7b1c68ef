"""Training path: gradients of the B200 layer against a plain PyTorch fp32
autograd reference of the same op (same routing decisions: the discrete top-K
is taken from the device; everything differentiable is recomputed in fp32).

Tolerance (bf16 activations/weights, fp32 accumulation): max|err| / max|ref|
<= 2e-2 for dx and every weight gradient."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 2e-2


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_16947_b200 as P

    return P


def _reference_grads(layer, x, dout, topk_idx):
    E, K = layer.E, layer.K
    xr = x.float().requires_grad_()
    wg = layer.wg[:E].float().requires_grad_()
    w1 = layer.w1.float().requires_grad_()
    w3 = layer.w3.float().requires_grad_()
    w2 = layer.w2.float().requires_grad_()
    idx = topk_idx.long()
    logits = xr @ wg.T
    w = torch.softmax(logits.gather(1, idx), dim=1)
    out = torch.zeros_like(xr)
    for k in range(K):
        yk = torch.zeros_like(xr)
        for e in idx[:, k].unique().tolist():
            sel = (idx[:, k] == e).nonzero().flatten()
            xs = xr[sel]
            h = torch.nn.functional.silu(xs @ w1[e].T) * (xs @ w3[e].T)
            yk = yk.index_add(0, sel, h @ w2[e].T)
        out = out + w[:, k:k + 1] * yk
    (out * dout.float()).sum().backward()
    return xr.grad, wg.grad, w1.grad, w3.grad, w2.grad


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-12)).item()


@pytest.mark.parametrize("G,E,K,d,F,T,s", [
    (4, 8, 2, 512, 1024, 2048, 1.0),
    (8, 32, 4, 256, 256, 1024, 1.5),
    (2, 8, 2, 256, 256, 512, 0.0),
])
def test_layer_gradients_match_fp32_reference(P, G, E, K, d, F, T, s):
    from paper_2511_16947_b200.layer import interleave_w13

    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
    layer = P.MoELayer(pl, d, F, K, seed=2, gate_bias=bias, train=True)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    layer(x)
    dx, dwg, dw13, dw2 = layer.backward_step(x, dout)
    torch.cuda.synchronize()
    layer.check_status()
    b = layer.buffers(T)
    rdx, rwg, rw1, rw3, rw2 = _reference_grads(layer, x, dout, b.topk_idx)
    assert _rel(dx, rdx) <= TOL, _rel(dx, rdx)
    assert _rel(dwg, rwg) <= TOL, _rel(dwg, rwg)
    assert _rel(dw2, rw2) <= TOL, _rel(dw2, rw2)
    assert _rel(dw13, interleave_w13(rw1, rw3)) <= TOL, _rel(dw13, interleave_w13(rw1, rw3))
    # deterministic (no float atomics)
    layer(x)
    dx2, dwg2, dw132, dw22 = layer.backward_step(x, dout)
    assert torch.equal(dx, dx2) and torch.equal(dw13, dw132) and torch.equal(dw2, dw22) and torch.equal(dwg, dwg2)


def test_autograd_function(P):
    from paper_2511_16947_b200.layer import MoEFunction

    pl = P.cayley_symmetric(P.ClusterShape(4, 8, 2))
    layer = P.MoELayer(pl, 256, 256, 2, seed=1, train=True)
    wg = torch.nn.Parameter(layer.wg)
    w13 = torch.nn.Parameter(layer.w13)
    w2 = torch.nn.Parameter(layer.w2)
    x = torch.randn(512, 256, device="cuda").to(torch.bfloat16).requires_grad_()
    out = MoEFunction.apply(x, wg, w13, w2, layer)
    out.float().square().mean().backward()
    assert x.grad.shape == x.shape and torch.isfinite(x.grad.float()).all()
    assert w13.grad.shape == w13.shape and w2.grad.shape == w2.shape and wg.grad.shape == wg.shape
    assert w13.grad.float().abs().sum() > 0 and wg.grad[:8].float().abs().sum() > 0


def test_backward_pair_and_single_cta_agree(P, tune):
    """The backward GEMMs (SwiGLU dgrad, dX dgrad, K-ragged weight gradients) on the
    CTA-pair kernel (256-row tiles, MN-major operand halves) and on the 1-CTA kernel:
    both within tolerance of fp32 autograd and identical bit for bit (same K order)."""
    from paper_2511_16947_b200.layer import interleave_w13

    G, E, K, d, F, T, s = 4, 8, 2, 512, 1024, 4096, 1.0
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    g = torch.Generator(device="cuda").manual_seed(19)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    res = {}
    for pair in ("0", "1"):
        tune(ffn_pair=int(pair))
        layer = P.MoELayer(pl, d, F, K, seed=2, gate_bias=bias, train=True)
        layer(x)
        res[pair] = [t.clone() for t in layer.backward_step(x, dout)]
        torch.cuda.synchronize()
        layer.check_status()
    rdx, rwg, rw1, rw3, rw2 = _reference_grads(layer, x, dout, layer.buffers(T).topk_idx)
    for pair in ("0", "1"):
        dx, dwg, dw13, dw2 = res[pair]
        assert _rel(dx, rdx) <= TOL and _rel(dw2, rw2) <= TOL and _rel(dw13, interleave_w13(rw1, rw3)) <= TOL
    for a, b in zip(res["0"], res["1"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("pair", ["0", "1"])
def test_store_and_copy_widths_agree(P, tune, pair):
    """256-bit epilogue stores / pre-activation loads (hep_tuning.st256) and the 256-bit
    permute (hep_tuning.lsu256) against their 128-bit fallbacks (taken for unaligned rows and
    peer-row destinations): forward output and all gradients identical bit for bit."""
    G, E, K, d, F, T, s = 4, 8, 2, 512, 1024, 4096, 1.0
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    g = torch.Generator(device="cuda").manual_seed(23)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    tune(ffn_pair=int(pair))
    res = {}
    for wide in ("0", "1"):
        tune(st256=int(wide))
        tune(lsu256=int(wide))
        layer = P.MoELayer(pl, d, F, K, seed=2, gate_bias=bias, train=True)
        y = layer(x).clone()
        b = layer.buffers(T)
        res[wide] = [y, b.rows.clone()] + [t.clone() for t in layer.backward_step(x, dout)]
        torch.cuda.synchronize()
        layer.check_status()
    for a, b in zip(res["0"], res["1"]):
        assert torch.equal(a, b)


def test_backward_light_expert_split(P, tune):
    """CTA-pair backward with the light experts' dgrad tiles on the 1-CTA kernel
    (hep_tuning.ffn_light_rows): gradients identical bit for bit to the unsplit backward."""
    G, E, K, d, F, T, s = 4, 64, 4, 256, 256, 8192, 1.5  # Cayley (p=2, q=5); R / E = 512 -> pairs
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    g = torch.Generator(device="cuda").manual_seed(29)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    tune(ffn_pair=1)
    from paper_2511_16947_b200 import _lib

    res = {}
    for lr in ("0", "256"):
        tune(ffn_light_rows=int(lr))
        assert int(_lib.lib().hep_moe_ffn_bwd_launches(T * K, E)) == (9 if lr == "0" else 13)
        layer = P.MoELayer(pl, d, F, K, seed=3, gate_bias=bias, train=True)
        y = layer(x).clone()
        res[lr] = [y] + [t.clone() for t in layer.backward_step(x, dout)]
        torch.cuda.synchronize()
        layer.check_status()
    loads = layer.expert_loads(T)
    assert min(loads) <= 256 < max(loads)  # both lists are populated
    for a, b in zip(res["0"], res["256"]):
        assert torch.equal(a, b)


def test_backward_wgrad_expert_order(P, tune):
    """Weight-gradient tiles visited heaviest expert first (hep_tuning.wgrad_order) or in
    expert order: every output tile is one CTA's K-ordered sum, so the bits match."""
    G, E, K, d, F, T, s = 4, 64, 4, 256, 256, 8192, 1.5
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    g = torch.Generator(device="cuda").manual_seed(31)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    res = {}
    for pair in ("0", "1"):
        tune(ffn_pair=int(pair))
        for order in ("0", "1"):
            tune(wgrad_order=int(order))
            layer = P.MoELayer(pl, d, F, K, seed=4, gate_bias=bias, train=True)
            layer(x)
            res[pair + order] = [t.clone() for t in layer.backward_step(x, dout)]
            torch.cuda.synchronize()
            layer.check_status()
    for key in ("01", "10", "11"):
        for a, b in zip(res["00"], res[key]):
            assert torch.equal(a, b), key
