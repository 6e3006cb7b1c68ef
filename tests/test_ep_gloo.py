"""World-size-2 gloo test (CPU) of the EP collectives: DistComm (one process
per rank over torch.distributed) must deliver exactly what LocalComm computes
for the histogram all-gather and the uneven all-to-all-v dispatch / combine."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(world, E=6, d=5, seed=0):
    g = torch.Generator().manual_seed(seed)
    hist = [torch.randint(0, 100, (1, E), generator=g, dtype=torch.int64) for _ in range(world)]
    send_counts = [[int(v) for v in torch.randint(0, 7, (world,), generator=g)] for _ in range(world)]
    recv_counts = [[send_counts[s][r] for s in range(world)] for r in range(world)]
    sends = [torch.randn(sum(send_counts[r]), d, generator=g) for r in range(world)]
    return hist, send_counts, recv_counts, sends


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_16947_b200.ep import DistComm, LocalComm

        hist, sc, rc, sends = _inputs(world)
        ref_h = LocalComm(world).all_gather(hist)[rank]
        ref_r = LocalComm(world).all_to_all(sends, sc, rc)[rank]
        ref_back = LocalComm(world).all_to_all(LocalComm(world).all_to_all(sends, sc, rc), rc, sc)[rank]
        comm = DistComm()
        got_h = comm.all_gather([hist[rank]])[0]
        got_r = comm.all_to_all([sends[rank]], [sc[rank]], [rc[rank]])[0]
        got_back = comm.all_to_all([got_r], [rc[rank]], [sc[rank]])[0]
        ok = torch.equal(got_h, ref_h) and torch.equal(got_r, ref_r) and torch.equal(got_back, ref_back)
        ok = ok and torch.equal(got_back, sends[rank])  # combine returns rows to their send positions
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_comm_matches_local_comm(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _grads(world, E, seed):
    from paper_2511_16947_b200.core import ClusterShape
    from paper_2511_16947_b200.placement import greedy_replica_counts, monte_carlo_placement

    shape = ClusterShape(world, E, 2)
    loads = [(e * 37) % 11 + 1 for e in range(E)]
    pl = monte_carlo_placement(loads, greedy_replica_counts(loads, 2 * E, max_count=world), shape, 8, seed)
    n_slots = max(max(pl.slots[e] for e in h) + 1 if h else 1 for h in pl.hosted)
    g = torch.Generator().manual_seed(seed)
    dw13 = [torch.randn(n_slots, 4, 3, generator=g) for _ in range(world)]
    dw2 = [torch.randn(n_slots, 3, 2, generator=g) for _ in range(world)]
    return pl, dw13, dw2


def _edp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_16947_b200.ep import DistComm, LocalComm, edp_reduce

        pl, dw13, dw2 = _grads(world, 6, 3)
        # expected: sum over the replicas of each expert, identical on every replica
        exp13 = {e: sum(dw13[r][pl.slots[e]] for r in sorted(set(pl.edp_groups[e]))) for e in range(pl.num_experts)}
        exp2 = {e: sum(dw2[r][pl.slots[e]] for r in sorted(set(pl.edp_groups[e]))) for e in range(pl.num_experts)}
        loc13, loc2 = [t.clone() for t in dw13], [t.clone() for t in dw2]
        edp_reduce(pl, LocalComm(world), list(range(world)), loc13, loc2)
        mine13, mine2 = dw13[rank].clone(), dw2[rank].clone()
        edp_reduce(pl, DistComm(), [rank], [mine13], [mine2])
        ok = torch.equal(mine13, loc13[rank]) and torch.equal(mine2, loc2[rank])
        for e in pl.hosted[rank]:
            sl = pl.slots[e]
            ok = ok and torch.allclose(mine13[sl], exp13[e]) and torch.allclose(mine2[sl], exp2[e])
        red = torch.full((3,), float(rank + 1))
        DistComm().all_reduce([red])
        ok = ok and torch.equal(red, torch.full((3,), float(world * (world + 1) // 2)))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_edp_gradient_reduction_over_gloo(world):
    """The expert-gradient reduction inside each EDP group (one all-to-all-v of the
    shared experts' gradients) gives, on every replica, the sum over the replicas
    — the same bits as the single-process LocalComm run."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_edp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _mig_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_16947_b200.core import ClusterShape
        from paper_2511_16947_b200.ep import DistComm, migrate_weights
        from paper_2511_16947_b200.placement import greedy_replica_counts, monte_carlo_placement, random_placement

        E = 6
        shape = ClusterShape(world, E, 2)
        old = random_placement(shape, 1)
        loads = [40, 1, 1, 9, 3, 2]
        new = monte_carlo_placement(loads, greedy_replica_counts(loads, 2 * E, max_count=world), shape, 8, 2)

        def nslots(pl, r):
            return max([pl.slots[e] + 1 for e in pl.hosted[r]] + [1])

        def expert_w(e):  # every replica of expert e holds the same weights
            g = torch.Generator().manual_seed(100 + e)
            return torch.randn(4, 3, generator=g), torch.randn(3, 2, generator=g)

        w13 = torch.zeros(nslots(old, rank), 4, 3)
        w2 = torch.zeros(nslots(old, rank), 3, 2)
        for e in old.hosted[rank]:
            w13[old.slots[e]], w2[old.slots[e]] = expert_w(e)
        n13 = torch.full((nslots(new, rank), 4, 3), float("nan"))
        n2 = torch.full((nslots(new, rank), 3, 2), float("nan"))
        st = migrate_weights(old, new, DistComm(), [rank], [w13], [w2], [n13], [n2])
        ok = True
        for e in new.hosted[rank]:
            a, b = expert_w(e)
            ok = ok and torch.equal(n13[new.slots[e]], a) and torch.equal(n2[new.slots[e]], b)
        pairs = lambda pl: {(e, g) for e, grp in enumerate(pl.edp_groups) for g in grp}  # noqa: E731
        ok = ok and st["moved_replicas"] == len(pairs(new) - pairs(old))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_weight_migration_over_gloo(world):
    """Adaptive replacement on real ranks: after migrate_weights every GPU holds
    exactly the experts of the new placement in the new slots, and the number of
    replicas moved equals the reference's changed_slots (adaptive.py:157)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mig_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res
