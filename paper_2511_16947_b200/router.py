"""Token-range routing and all-to-all accounting on the GPU (drop-in API).

Same public surface as the reference ``harmonyep.router``
(``/root/reference/pkg/src/harmonyep/router.py``):

  RoutingTable          :38-60   ranges (expert, src, dst, count); ``to_csv`` is the
                                 byte-level identity format (acceptance C8)
  TransferPlan          :63-94
  route_tokens          :161-163 (Algorithm 1, locality first)
  route_topology_aware  :166-175 (same node before cross node)
  build_transfer_plan   :178-226

Routing and aggregation run in the scheduler kernel (``csrc/sched.cu``) via
``hep_sched_route`` / ``hep_transfer_plan``; the host keeps only the
reference's cheap metadata checks (plan/placement identity, integrality —
``_check_plan`` :97-111), the per-expert sum and sign checks happen on the
device.
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ContractViolation, DimensionError, LoadMatrix, Placement, ReplicaLoadPlan, Topology
from .scheduler import HEP_SCHED_TOPO, MAX_GPUS, CapacityError, device_scheduler


@dataclass(frozen=True)
class RoutingTable:
    """Ordered (expert, src GPU, dst GPU, token_count) ranges; for a fixed
    (expert, src) they partition that source's tokens in sequence order."""

    ranges: tuple[tuple[int, int, int, int], ...]

    def to_csv(self) -> str:
        out = io.StringIO()
        out.write("expert,src,dst,count\n")
        out.writelines(f"{e},{s},{d},{c}\n" for e, s, d, c in self.ranges)
        return out.getvalue()

    def local_volume(self) -> int:
        return sum(c for _, s, d, c in self.ranges if s == d)

    def total_volume(self) -> int:
        return sum(r[3] for r in self.ranges)


@dataclass(frozen=True)
class TransferPlan:
    """Pairwise all-to-all token counts; the diagonal is local traffic."""

    pair_counts: tuple[tuple[int, ...], ...]
    send: tuple[int, ...]
    recv: tuple[int, ...]
    local: tuple[int, ...]
    send_intra: tuple[int, ...]
    recv_intra: tuple[int, ...]
    send_inter: tuple[int, ...]
    recv_inter: tuple[int, ...]
    intra_volume: int
    inter_volume: int

    @property
    def local_volume(self) -> int:
        return sum(self.local)

    def max_intra(self) -> int:
        return max((max(a, b) for a, b in zip(self.send_intra, self.recv_intra)), default=0)

    def max_inter(self) -> int:
        return max((max(a, b) for a, b in zip(self.send_inter, self.recv_inter)), default=0)

    @classmethod
    def from_flat(cls, G: int, flat) -> "TransferPlan":
        """Decode the ``d_transfer`` layout of include/hep.h."""
        v = [int(x) for x in flat]
        pair = tuple(tuple(v[i * G:(i + 1) * G]) for i in range(G))
        k = G * G
        vec = [tuple(v[k + i * G: k + (i + 1) * G]) for i in range(7)]
        return cls(pair, *vec, intra_volume=v[k + 7 * G], inter_volume=v[k + 7 * G + 1])


def _check_plan_host(placement: Placement, loads: LoadMatrix, plan: ReplicaLoadPlan) -> None:
    if not plan.matches_placement(placement):
        raise ContractViolation("plan was not solved against this placement")
    if (loads.num_experts, loads.num_gpus) != (placement.num_experts, placement.num_gpus):
        raise DimensionError("loads do not match placement")
    if not plan.is_integral():
        raise ContractViolation("plan must be integerized before routing")


def _route(placement: Placement, loads: LoadMatrix, plan: ReplicaLoadPlan, topology: Topology | None) -> RoutingTable:
    import torch

    _check_plan_host(placement, loads, plan)
    gpn = topology.gpus_per_node if topology is not None else 0
    dev = device_scheduler(placement, gpn)
    G = placement.num_gpus
    xi = np.fromiter((int(v) for row in plan.entries for v in row), dtype=np.int64)
    d_xi = torch.as_tensor(xi if xi.size else np.zeros(1, np.int64)).to(dev.device)
    d_loads = torch.as_tensor(loads.as_array()).to(dev.device)
    flags = HEP_SCHED_TOPO if (topology is not None and topology.num_nodes > 1) else 0
    dev.launch_route(d_loads, G, 1, d_xi, flags)
    dev.check_status("route_tokens")
    return RoutingTable(dev.host_ranges())


def route_tokens(placement: Placement, loads: LoadMatrix, plan: ReplicaLoadPlan) -> RoutingTable:
    """Algorithm 1 (locality-first greedy) on the device."""
    return _route(placement, loads, plan, None)


def route_topology_aware(placement: Placement, loads: LoadMatrix, plan: ReplicaLoadPlan,
                         topology: Topology) -> RoutingTable:
    """Same GPU, then same node, then cross node; identical to
    :func:`route_tokens` on a single node."""
    if topology.num_gpus != placement.num_gpus:
        raise DimensionError("topology does not match placement")
    return _route(placement, loads, plan, topology)


def build_transfer_plan(table: RoutingTable, topology: Topology) -> TransferPlan:
    """Aggregate a routing table into pairwise/send/recv/local volumes (device)."""
    torch = _lib.require_cuda()
    G = topology.num_gpus
    if G > MAX_GPUS:
        raise CapacityError(f"device transfer plan handles up to {MAX_GPUS} GPUs")
    n = len(table.ranges)
    arr = np.asarray(table.ranges, dtype=np.int64).reshape(n, 4) if n else np.zeros((1, 4), np.int64)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_ranges = torch.as_tensor(arr).to(dev)
    d_t = torch.zeros(G * G + 8 * G + 2, dtype=torch.int64, device=dev)
    d_st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(
        _lib.lib().hep_transfer_plan(G, topology.gpus_per_node, d_ranges.data_ptr(), n, d_t.data_ptr(),
                                     d_st.data_ptr(), _lib.stream_handle()),
        "hep_transfer_plan",
    )
    _lib.raise_status(int(d_st.item()), "build_transfer_plan")
    return TransferPlan.from_flat(G, d_t.cpu().tolist())
