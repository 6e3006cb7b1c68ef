"""Failure paths of the device pipeline: a micro-batch the scheduler
rejects, or whose schedule would overflow a rank's fixed NVLink receive buffer,
must raise the reference exception class from ``check_status`` without any
out-of-bounds access (the kernels queued behind the failing one see an empty
plan), and the layer must work again on the next valid micro-batch."""

import math
from fractions import Fraction

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_16947_b200 as P

    return P


def test_scheduler_error_leaves_empty_plan(P):
    """Expert 0 has no replica and receives tokens -> PlacementError (reference
    scheduler.py:344-347).  The assignment falls back to the identity row map, no
    FFN tiles run, nothing faults; the next micro-batch without expert-0 tokens
    is scheduled normally."""
    from paper_2511_16947_b200.core import PlacementError

    G, E, K, d, F, T = 4, 8, 2, 256, 256, 2048
    base = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    groups = ((),) + tuple(base.edp_groups[1:])
    pl = P.Placement(G, groups, base.slots)
    bias = torch.zeros(E)
    bias[0] = 30.0  # every token picks expert 0
    layer = P.MoELayer(pl, d, F, K, seed=1, gate_bias=bias)
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(3), device="cuda").to(torch.bfloat16)
    layer(x)
    torch.cuda.synchronize()  # no fault
    with pytest.raises(PlacementError):
        layer.check_status()
    b = layer.buffers(T)
    assert torch.equal(b.tok_row.view(-1).cpu(), torch.arange(T * K, dtype=torch.int32))
    assert int(layer.sched.n_ranges.item()) == 0 and int(layer.sched.gpu_load.sum().item()) == 0
    assert int(b.seg[:, 1].sum().item()) == 0
    # recovery: route around expert 0
    layer.gate_bias[0] = -30.0
    out = layer(x)
    torch.cuda.synchronize()
    layer.check_status()
    assert torch.isfinite(out.float()).all()
    assert int(b.hist[:, 0].sum().item()) == 0


def test_p2p_receive_capacity_overflow_raises(P):
    """NVLink path with receive buffers smaller than the balanced load: every rank
    detects the overflow on the identical plan, nothing is stored into the peers'
    buffers, CapacityError is raised; with the default capacity the same batch runs."""
    from paper_2511_16947_b200.core import CapacityError
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    G, E, K, d, F, T = 4, 8, 2, 256, 256, 4096
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(4), device="cuda").to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    small = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=2, gate_bias=bias, exchange="p2p",
                       recv_capacity_factor=0.5)
    assert small.ranks[0].p2p_buffers(small, T // G)["cap"] == math.ceil(0.5 * (T // G) * K)
    small.forward(xs)
    torch.cuda.synchronize()
    with pytest.raises(CapacityError):
        small.check_status()
    for rk in small.ranks:
        assert int(rk.bufs[T // G]["counts"].sum().item()) == 0
    ok = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=2, gate_bias=bias, exchange="p2p")
    outs = ok.forward(xs)
    torch.cuda.synchronize()
    ok.check_status()
    ref = P.MoELayer(pl, d, F, K, seed=2, gate_bias=bias)(x)
    assert torch.equal(torch.cat(outs, dim=0), ref)


def test_p2p_rejects_unequal_token_counts(P):
    from paper_2511_16947_b200.ep import EPMoELayer, LocalComm

    G, E, K, d, F = 2, 8, 2, 256, 256
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=2, exchange="p2p")
    xs = [torch.randn(256, d, device="cuda").to(torch.bfloat16), torch.randn(128, d, device="cuda").to(torch.bfloat16)]
    with pytest.raises(ValueError, match="same token count"):
        ep.forward(xs)


def _ref_integerize(groups, entries):
    """The reference's integerize_plan (scheduler.py:697-735), restated for the check."""
    out = []
    for group, row in zip(groups, entries):
        exact = [Fraction(v) for v in row]
        total = round(sum(exact))
        floors = [math.floor(v) for v in exact]
        units = total - sum(floors)
        rem = sorted(range(len(row)), key=lambda i: (-(exact[i] - floors[i]), group[i]))
        o = list(floors)
        for i in rem[:units]:
            o[i] += 1
        out.append(tuple(o))
    return tuple(out)


def test_integerize_float_plan_with_wide_magnitudes(P):
    """Float entries whose exact common denominator overflows int64:
    integerized on the device on a binary fixed point, same answer as the reference."""
    groups = ((0, 1), (1, 2), (2, 0))
    entries = ((1000.1, 0.9), (0.25, 2.75), (3e-12, 5.0 - 3e-12))
    plan = P.ReplicaLoadPlan(num_gpus=3, groups=groups, entries=entries, objective=0)
    got = P.integerize_plan(plan)
    assert got.entries == _ref_integerize(groups, entries)


def test_host_pipeline_ticket_lifetime(P):
    from paper_2511_16947_b200.layer import HostPipeline

    G, E, K, d, F, T = 4, 8, 2, 256, 256, 1024
    layer = P.MoELayer(P.cayley_symmetric(P.ClusterShape(G, E, 2)), d, F, K, seed=1)
    pipe = HostPipeline(layer, T, depth=2)
    xh = torch.randn(T, d).to(torch.bfloat16).pin_memory()
    t0 = pipe.submit(xh)
    first = pipe.result(t0, copy=True)
    pipe.submit(xh)
    pipe.submit(xh)
    with pytest.raises(RuntimeError, match="reused"):
        pipe.result(t0)
    assert torch.equal(pipe.result(2), first)
