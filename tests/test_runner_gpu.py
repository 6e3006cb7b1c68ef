"""LayerRunner: the reference's run_strategy loop (simulator.py:346-476) driving the
real device layer — periodic adaptive replacement inside the loop and
per-micro-batch MicrobatchMetrics rows from the device's own plans."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_16947_b200 as P

    return P


def test_runner_adaptive_replacement_and_metrics(P):
    from oracle import oracle as O
    from paper_2511_16947_b200.adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace
    from paper_2511_16947_b200.runner import LayerRunner
    from paper_2511_16947_b200.sweep import METRICS_CSV_HEADER

    G, E, K, d, F, T = 8, 8, 2, 256, 256, 4096
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, 1.5, 0))
    layer = P.MoELayer(pl, d, F, K, seed=1, gate_bias=bias)
    policy = ReplacementPolicy(check_interval=4, threshold=1.1, window=4, mc_samples=50)
    runner = LayerRunner(layer, policy, shape=shape)
    xs = [torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(s), device="cuda").to(torch.bfloat16)
          for s in range(10)]
    loads_seen, hists = [], []
    for i, x in enumerate(xs):
        runner.step(x)
        b = layer.buffers(T)
        h = b.hist.clone()
        torch.cuda.synchronize()
        layer.check_status()
        hists.append(h.cpu().numpy())
        loads_seen.append(h.sum(dim=0).cpu().tolist())
    # the check ran before micro-batch 4 and 8, on the window of the 4 previous micro-batches
    hist = LoadHistory(4)
    for v in loads_seen[:4]:
        hist.push(v)
    dec = evaluate_and_maybe_replace(pl, hist, policy, shape, 0)
    assert dec.replaced  # s = 1.5 on the 8-cycle is far from balanced
    assert runner.events and runner.events[0]["iteration"] == 4
    assert runner.placements[1][1] == dec.placement
    rows = runner.metrics()
    assert [r.index for r in rows] == list(range(10))
    placement_at = lambda i: [p for j, p in runner.placements if j <= i][-1]  # noqa: E731
    for i, r in enumerate(rows):
        ref = O.full_path(G, [tuple(g) for g in placement_at(i).edp_groups], hists[i].T.copy())
        assert r.max_gpu_load == max(ref["gpu_load"])
        assert r.a2a_intra == ref["intra"] and r.a2a_inter == ref["inter"]
        assert r.local_volume == sum(ref["local"])
        assert r.layer_time > 0
    assert max(r.balance_ratio for r in rows[4:]) < max(r.balance_ratio for r in rows[:4])
    csv = runner.metrics_csv("harmony", 1.5, 0)
    assert csv.splitlines()[0] == METRICS_CSV_HEADER and len(csv.splitlines()) == 11
