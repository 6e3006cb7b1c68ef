"""Expert-parallel protocol on one B200: all G ranks in one process
(LocalComm), each with its own scheduler handle, local expert-weight slots,
send/receive buffers and kernels, exchanging rows through the same
all-gather / all-to-all-v split sizes NCCL would use.  The result must be
bit-identical to the simulated-EP MoELayer (same tokens, weights, schedule)."""

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


def _placement(P, G, E, kind, s, seed=0):
    shape = P.ClusterShape(G, E, 2)
    if kind == "cayley":
        return P.cayley_symmetric(shape)
    from paper_2511_16947_b200.placement import greedy_replica_counts, monte_carlo_placement

    wl = P.gen_zipf_workload(shape, s, 2048, 1, seed)
    totals = wl.micro_batches[0].expert_totals()
    return monte_carlo_placement(totals, greedy_replica_counts(totals, 2 * E, max_count=G), shape, 20, seed)


@pytest.mark.parametrize("G,E,K,d,F,T,kind,s", [
    (4, 8, 2, 512, 1024, 4096, "cayley", 1.0),
    (8, 8, 2, 1024, 512, 8192, "asym", 1.5),
    (8, 128, 8, 512, 256, 8192, "cayley", 1.0),
    (8, 32, 4, 256, 256, 4096, "asym", 2.0),
    (2, 8, 2, 256, 128, 2048, "cayley", 0.0),
])
def test_local_ep_matches_simulated_layer(P, G, E, K, d, F, T, kind, s):
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    pl = _placement(P, G, E, kind, s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
    sim = P.MoELayer(pl, d, F, K, seed=3, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(5), device="cuda").to(torch.bfloat16)
    ref = sim(x).clone()
    ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=3, gate_bias=bias)
    tps = T // G
    outs = ep.forward([x[r * tps:(r + 1) * tps].contiguous() for r in range(G)])
    torch.cuda.synchronize()
    sim.check_status()
    for rk in ep.ranks:
        rk.sched.check_status("ep")
    got = torch.cat(outs, dim=0)
    assert torch.equal(got, ref), (got.float() - ref.float()).abs().max().item()
    # every rank computed the identical schedule
    x0 = ep.ranks[0].sched
    for rk in ep.ranks[1:]:
        assert torch.equal(rk.sched.xi, x0.xi) and torch.equal(rk.sched.ranges, x0.ranges)


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-12)).item()


@pytest.mark.parametrize("G,E,K,d,F,T,kind,s", [
    (4, 8, 2, 512, 512, 4096, "cayley", 1.0),
    (8, 32, 4, 256, 256, 4096, "asym", 1.5),
    (2, 8, 2, 256, 256, 1024, "cayley", 0.0),
])
def test_local_ep_backward_matches_simulated_layer(P, G, E, K, d, F, T, kind, s):
    """EP training: forward and dx bit-identical to the simulated layer (rows are
    independent in every GEMM); router and expert weight gradients equal to the
    simulated layer's up to fp32 summation order (the EP sums per-replica
    partials); all replicas of an expert hold bit-identical gradients after the
    EDP-group reduction."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    pl = _placement(P, G, E, kind, s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
    sim = P.MoELayer(pl, d, F, K, seed=4, gate_bias=bias, train=True)
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    ref = sim(x).clone()
    rdx, rdwg, rdw13, rdw2 = sim.backward_step(x, dout)
    ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=4, gate_bias=bias, train=True)
    tps = T // G
    xs = [x[r * tps:(r + 1) * tps].contiguous() for r in range(G)]
    outs = ep.forward(xs)
    got = torch.cat([o.clone() for o in outs], dim=0)
    grads = ep.backward([dout[r * tps:(r + 1) * tps].contiguous() for r in range(G)])
    torch.cuda.synchronize()
    sim.check_status()
    for rk in ep.ranks:
        rk.sched.check_status("ep")
    assert torch.equal(got, ref)
    dx = torch.cat([gr[0] for gr in grads], dim=0)
    assert torch.equal(dx, rdx), _rel(dx, rdx)
    for gr in grads:
        assert _rel(gr[1], rdwg) <= 1e-3
        assert torch.equal(gr[1], grads[0][1])
    for e in range(E):
        members = sorted(set(pl.edp_groups[e]))
        sl = pl.slots[e]
        for q in members:
            assert _rel(grads[q][2][sl], rdw13[e]) <= 1e-3, (e, q)
            assert _rel(grads[q][3][sl], rdw2[e]) <= 1e-3, (e, q)
            assert torch.equal(grads[q][2][sl], grads[members[0]][2][sl])
            assert torch.equal(grads[q][3][sl], grads[members[0]][3][sl])


def test_local_ep_weight_migration(P):
    """Cayley -> adaptive placement by moving weights between the ranks' slots:
    the migrated layer's outputs are bit-identical to a layer built directly on
    the new placement, and the moved replicas equal the reference's changed_slots."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    G, E, K, d, F, T = 8, 16, 2, 256, 256, 4096
    old = _placement(P, G, E, "cayley", 1.5)
    new = _placement(P, G, E, "asym", 1.5, seed=1)
    bias = torch.tensor(P.zipf_gate_bias(E, 1.5, 0))
    ep = EPMoELayer(old, d, F, K, LocalComm(G), range(G), seed=2, gate_bias=bias)
    st = ep.migrate(new)
    fresh = EPMoELayer(new, d, F, K, LocalComm(G), range(G), seed=2, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(4), device="cuda").to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    got = torch.cat([o.clone() for o in ep.forward(xs)])
    ref = torch.cat([o.clone() for o in fresh.forward(xs)])
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    for a, b in zip(ep.ranks, fresh.ranks):
        assert torch.equal(a.w13, b.w13) and torch.equal(a.w2, b.w2)
    pairs = lambda pl: {(e, g) for e, grp in enumerate(pl.edp_groups) for g in grp}  # noqa: E731
    assert st["moved_replicas"] == len(pairs(new) - pairs(old)) > 0


@pytest.mark.parametrize("G,E,K,d,F,T,kind,s", [
    (4, 8, 2, 512, 512, 4096, "cayley", 1.0),
    (8, 32, 4, 256, 256, 4096, "asym", 1.5),
    (8, 128, 8, 256, 256, 8192, "cayley", 1.0),
])
def test_local_ep_p2p_exchange_matches_collectives(P, G, E, K, d, F, T, kind, s):
    """Both exchanges as peer-memory stores (dispatch kernel into the destination's
    receive buffer, down-projection epilogue into the source's return buffer) give
    the same bits as the all-to-all-v collectives and as the single-device layer."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    pl = _placement(P, G, E, kind, s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(11), device="cuda").to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    a = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=bias)
    b = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=bias, exchange="p2p")
    ref = torch.cat([o.clone() for o in a.forward(xs)])
    got = torch.cat([o.clone() for o in b.forward(xs)])
    got2 = torch.cat([o.clone() for o in b.forward(xs)])  # buffers reused across micro-batches
    # both exchanges without the per-slot regrouping of the received rows
    c = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=bias, exchange="p2p")
    c.regroup_rows = False
    a.regroup_rows = False
    got3 = torch.cat([o.clone() for o in c.forward(xs)])
    ref3 = torch.cat([o.clone() for o in a.forward(xs)])
    b.regroup_rows = False  # toggled after the buffers exist
    got4 = torch.cat([o.clone() for o in b.forward(xs)])
    torch.cuda.synchronize()
    for rk in b.ranks:
        rk.sched.check_status("p2p")
    assert torch.equal(got, ref)
    assert torch.equal(got2, ref)
    assert torch.equal(got3, ref) and torch.equal(ref3, ref) and torch.equal(got4, ref)
    sim = P.MoELayer(pl, d, F, K, seed=6, gate_bias=bias)
    assert torch.equal(sim(x), ref)


def test_local_ep_p2p_light_split_on_pairs(P, tune):
    """CTA pairs forced, so every rank's FFN splits its light slots onto the 1-CTA
    kernel: the peer-row (NVLink store) epilogue of both kernels, the collectives
    path and the single-device layer agree bit for bit."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    tune(ffn_pair=1)
    G, E, K, d, F, T, s = 8, 128, 8, 256, 256, 8192, 1.5
    pl = _placement(P, G, E, "cayley", s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(12), device="cuda").to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    a = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=bias)
    b = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=bias, exchange="p2p")
    ref = torch.cat([o.clone() for o in a.forward(xs)])
    got = torch.cat([o.clone() for o in b.forward(xs)])
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    sim = P.MoELayer(pl, d, F, K, seed=6, gate_bias=bias)
    assert torch.equal(sim(x), ref)
    assert int(P._lib.lib().hep_moe_ffn_launches(T * K, E, 0)) == 8


def _p2p_worker(rank, world, port, q, kind="cayley"):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_16947_b200 as P
        from paper_2511_16947_b200.ep import DistComm, EPMoELayer

        G, E, K, d, F, T = world, 8, 2, 256, 256, 2048
        pl = _placement(P, G, E, kind, 1.5)
        bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
        x = torch.randn(G * T, d, generator=torch.Generator(device="cuda").manual_seed(12), device="cuda")
        x = x.to(torch.bfloat16)[rank * T:(rank + 1) * T].contiguous()
        layer = EPMoELayer(pl, d, F, K, DistComm(), [rank], seed=7, gate_bias=bias, exchange="p2p")
        outs = [layer.forward([x])[0].clone() for _ in range(2)]
        torch.cuda.synchronize()
        # the device-synchronised step has no host sync: capture it as a CUDA graph and replay
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        dist.barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            out_g = layer.forward([x], stream=side)[0]
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        layer.check_sync()
        q.put((rank, outs[0].float().cpu().numpy(), out_g.float().cpu().numpy()))  # pickled by value
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, repr(exc), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "cayley"), (4, "asym")])
def test_ep_p2p_over_cuda_ipc_processes(P, world, kind):
    """One process per rank (all on this GPU), peer buffers mapped with CUDA IPC and the
    ranks synchronised by device-side barriers: the NVLink-path forward — eager, and
    replayed from a CUDA graph — equals the in-process reference bit for bit; 2 ranks on
    the Cayley placement and 4 ranks on an asymmetric (adaptive) placement."""
    import socket

    import torch.multiprocessing as mp
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, o1, o2 = q.get(timeout=300)
        res[r] = (o1, o2)
    for p in procs:
        p.join(timeout=60)
    G, E, K, d, F, T = world, 8, 2, 256, 256, 2048
    pl = _placement(P, G, E, kind, 1.5)
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    x = torch.randn(G * T, d, generator=torch.Generator(device="cuda").manual_seed(12), device="cuda").to(torch.bfloat16)
    ref = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=7, gate_bias=bias).forward(
        [x[r * T:(r + 1) * T].contiguous() for r in range(G)])
    for r in range(world):
        o1, o2 = res[r]
        assert not isinstance(o1, str), o1
        want = ref[r].float().cpu().numpy()
        assert np.array_equal(o1, want) and np.array_equal(o2, want), r


@pytest.mark.parametrize("G,E,K,d,F,T,kind,s", [
    (4, 8, 2, 512, 512, 4096, "cayley", 1.0),
    (8, 32, 4, 256, 256, 4096, "asym", 1.5),
])
def test_local_ep_training_over_peer_stores(P, G, E, K, d, F, T, kind, s):
    """EP training with both directions of both exchanges as peer stores (dispatch kernel,
    FFN output rows and dX rows stored into the sources' buffers, dY rows into the
    destinations'): forward, dx and every gradient bit-identical to the NCCL-style
    all-to-all-v training path (the exchanges only move rows; the GEMM tiles are the same)."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    pl = _placement(P, G, E, kind, s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0))
    g = torch.Generator(device="cuda").manual_seed(31)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    tps = T // G
    xs = [x[r * tps:(r + 1) * tps].contiguous() for r in range(G)]
    ds = [dout[r * tps:(r + 1) * tps].contiguous() for r in range(G)]
    res = {}
    for exchange in ("nccl", "p2p"):
        ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=8, gate_bias=bias, train=True, exchange=exchange)
        outs = [o.clone() for o in ep.forward(xs)]
        grads = ep.backward(ds)
        torch.cuda.synchronize()
        ep.check_status()
        res[exchange] = (outs, grads)
    (o1, g1), (o2, g2) = res["nccl"], res["p2p"]
    for r in range(G):
        assert torch.equal(o1[r], o2[r]), r
        for a, b in zip(g1[r], g2[r]):
            assert torch.equal(a, b), r


def _p2p_train_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_16947_b200 as P
        from paper_2511_16947_b200.ep import DistComm, EPMoELayer

        G, E, K, d, F, T = world, 8, 2, 256, 256, 2048
        pl = _placement(P, G, E, "cayley", 1.0)
        bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
        g = torch.Generator(device="cuda").manual_seed(13)
        x = torch.randn(G * T, d, generator=g, device="cuda").to(torch.bfloat16)[rank * T:(rank + 1) * T].contiguous()
        dout = torch.randn(G * T, d, generator=g, device="cuda").to(torch.bfloat16)[rank * T:(rank + 1) * T].contiguous()
        layer = EPMoELayer(pl, d, F, K, DistComm(), [rank], seed=9, gate_bias=bias, train=True, exchange="p2p")
        out = layer.forward([x])[0].clone()
        dx, dwg, dw13, dw2 = layer.backward([dout])[0]
        torch.cuda.synchronize()
        layer.check_sync()
        layer.check_status()
        q.put((rank, [t.float().cpu().numpy() for t in (out, dx, dwg, dw13, dw2)]))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_ep_training_over_cuda_ipc_two_processes(P):
    """EP training with the NVLink exchanges between two real processes (CUDA IPC peer
    buffers, device-side barriers; the EDP gradient reduction and the router all-reduce
    over the process group): forward, dx and all gradients equal to the in-process
    LocalComm training step bit for bit."""
    import socket

    import torch.multiprocessing as mp
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    world = 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_train_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, v = q.get(timeout=300)
        res[r] = v
    for p in procs:
        p.join(timeout=60)
    G, E, K, d, F, T = world, 8, 2, 256, 256, 2048
    pl = _placement(P, G, E, "cayley", 1.0)
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    g = torch.Generator(device="cuda").manual_seed(13)
    x = torch.randn(G * T, d, generator=g, device="cuda").to(torch.bfloat16)
    dout = torch.randn(G * T, d, generator=g, device="cuda").to(torch.bfloat16)
    ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=9, gate_bias=bias, train=True, exchange="p2p")
    outs = ep.forward([x[r * T:(r + 1) * T].contiguous() for r in range(G)])
    grads = ep.backward([dout[r * T:(r + 1) * T].contiguous() for r in range(G)])
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        want = [outs[r]] + list(grads[r])
        for got, ref in zip(res[r], want):
            assert np.array_equal(got, ref.float().cpu().numpy()), r


@pytest.mark.parametrize("G,E,K,d,F,T,kind,s,ratio", [
    (4, 8, 2, 512, 512, 4096, "cayley", 1.0, 0.5),
    (8, 32, 4, 256, 256, 4096, "asym", 1.5, 0.5),
    (8, 128, 8, 256, 256, 8192, "cayley", 1.0, 0.25),
    (2, 8, 2, 256, 128, 2048, "cayley", 0.0, 1.0),
])
def test_local_ep_pipelined_split(P, G, E, K, d, F, T, kind, s, ratio):
    """harmony_pipelined over the EP group: the static share's assignment, permute and
    all-to-all-v on a side stream while the scheduled share is solved; one FFN over both
    phases' received rows.  The outputs equal the plain EP layer and the single-device
    pipelined layer bit for bit, and every rank holds the same two-phase schedule as the
    single-device layer's (static plan, scheduled plan, GPU loads)."""
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    pl = _placement(P, G, E, kind, s)
    bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(13), device="cuda").to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    plain = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=5, gate_bias=bias)
    pipe = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=5, gate_bias=bias, pipeline_ratio=ratio)
    ref = torch.cat([o.clone() for o in plain.forward(xs)])
    got = torch.cat([o.clone() for o in pipe.forward(xs)])
    got2 = torch.cat([o.clone() for o in pipe.forward(xs)])  # buffers reused across micro-batches
    torch.cuda.synchronize()
    for rk in pipe.ranks:
        rk.sched.check_status("pipelined")
    assert torch.equal(got, ref), (got.float() - ref.float()).abs().max().item()
    assert torch.equal(got2, ref)
    sim = P.MoELayer(pl, d, F, K, seed=5, gate_bias=bias, pipeline_ratio=ratio)
    assert torch.equal(sim(x), ref)
    torch.cuda.synchronize()
    s0 = pipe.ranks[0].sched
    for rk in pipe.ranks:
        assert torch.equal(rk.sched.xi, sim.sched.xi) and torch.equal(rk.sched.ranges, sim.sched.ranges)
        assert torch.equal(rk.sched.split, sim.sched.split)
        assert torch.equal(rk.sched.former.xi, s0.former.xi)
