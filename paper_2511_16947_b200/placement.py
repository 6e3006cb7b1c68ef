"""Init-time placement constructors consumed by the MoE layer (host side).

Placements are built once, before training/serving, and uploaded to the
device scheduler; they are not on the per-micro-batch path.  Same names and
outputs as the reference (``/root/reference/pkg/src/harmonyep/placement.py``),
pinned by the reference's Cayley goldens (tests/golden/placements.json):

  cayley_symmetric      :207-265  catalogue: 8-cycle (p=3,q=1), 4x4 torus (4,2),
                                  K4,4 (3,2), complete graphs + XOR matchings (q >= p)
  identical_placement   :471-487  merged-EP layout (vanilla / merged_ep baselines)
  validate_placement    :490-528
  density_oracle        :111-187  (exact: zeta transform over GPU subsets)
  random / greedy_replica_counts / monte_carlo_placement / symmetric_placement
                        :358-468  (asymmetric layouts for adaptive replacement)
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .core import CapacityError, ClusterShape, ConstructionError, ContractViolation, DimensionError, Placement

SUPPORTED_CAYLEY = (
    "(p=3, q=1)  8 GPUs x  8 experts: cycle",
    "(p=4, q=2) 16 GPUs x 32 experts: 4x4 torus",
    "(p=3, q=2)  8 GPUs x 16 experts: K4,4",
    "(p, q>=p)  2^p GPUs x 2^(p+q-1) experts: complete graphs + matchings",
)


def _pow2(v: int) -> bool:
    return v > 0 and not v & (v - 1)


def _xor_matching_layout(p: int, q: int) -> Placement:
    """Whole copies of K_{2^p} (each 1-factorised into XOR matchings v<->v^c,
    c = 1..2^p-1) followed by the first residual matchings; one slot per
    matching, so slots are proper by construction."""
    n = 1 << p
    n_edges = 1 << (p + q - 1)
    per_copy = n * (n - 1) // 2
    copies, rest = divmod(n_edges, per_copy)
    if copies < 1 or rest % (n // 2):
        raise ConstructionError(f"(p={p}, q={q}) does not decompose into complete graphs plus matchings")
    matchings = [c for _ in range(copies) for c in range(1, n)] + list(range(1, rest // (n // 2) + 1))
    groups, slots = [], []
    for slot, c in enumerate(matchings):
        for v in range(n):
            w = v ^ c
            if v < w:
                groups.append((v, w))
                slots.append(slot)
    return Placement(n, tuple(groups), tuple(slots))


def cayley_symmetric(shape: ClusterShape) -> Placement:
    """Catalogued vertex-transitive d=2 placement for power-of-two shapes."""
    if shape.d != 2:
        raise ConstructionError(f"symmetric catalog requires d=2, got d={shape.d}; supported: {SUPPORTED_CAYLEY}")
    G, E = shape.num_gpus, shape.num_experts
    if not (_pow2(G) and _pow2(E)):
        raise ConstructionError(
            f"symmetric catalog requires powers of two, got {G} GPUs, {E} experts; supported: {SUPPORTED_CAYLEY}"
        )
    p = G.bit_length() - 1
    q = E.bit_length() - p  # E = 2^(p+q-1)
    if q < 1:
        raise ConstructionError(f"fewer experts than GPUs is not catalogued; supported: {SUPPORTED_CAYLEY}")
    if (p, q) == (3, 1):  # the 8-cycle, alternating slots
        return Placement(8, tuple((v, (v + 1) % 8) for v in range(8)), tuple(v % 2 for v in range(8)))
    if (p, q) == (4, 2):  # 4x4 torus: row cycles (slots 0/1), then column cycles (slots 2/3)
        groups, slots = [], []
        for x in range(4):
            for y in range(4):
                groups.append((4 * x + y, 4 * x + (y + 1) % 4))
                slots.append(y % 2)
        for x in range(4):
            for y in range(4):
                groups.append((4 * x + y, 4 * ((x + 1) % 4) + y))
                slots.append(2 + x % 2)
        return Placement(16, tuple(groups), tuple(slots))
    if (p, q) == (3, 2):  # K4,4 as two 4-cycles plus the cross cycle
        groups, slots = [], []
        for a in range(2):
            for b in range(4):
                groups.append((4 * a + b, 4 * a + (b + 1) % 4))
                slots.append(b % 2)
        for a in range(2):
            for b in range(4):
                groups.append((4 * a + b, 4 * (1 - a) + (b + 1) % 4))
                slots.append(2 + b % 2)
        return Placement(8, tuple(groups), tuple(slots))
    if q >= p:
        return _xor_matching_layout(p, q)
    raise ConstructionError(f"no catalogued construction for (p={p}, q={q}); supported: {SUPPORTED_CAYLEY}")


def identical_placement(shape: ClusterShape) -> Placement:
    """Every EP group places experts identically: expert e lives on EP rank
    e // (E/ep) of each of the d groups."""
    ep = shape.ep_degree
    if shape.num_experts % ep:
        raise ConstructionError(f"{shape.num_experts} experts do not spread evenly over EP degree {ep}")
    per_rank = shape.num_experts // ep
    groups = tuple(tuple(e // per_rank + k * ep for k in range(shape.d)) for e in range(shape.num_experts))
    return Placement(shape.num_gpus, groups, tuple(e % per_rank for e in range(shape.num_experts)))


def validate_placement(placement: Placement, shape: ClusterShape, uniform: bool = False) -> list[str]:
    """Every invariant violation (empty list = valid)."""
    out: list[str] = []
    if placement.num_experts != shape.num_experts:
        out.append(f"expert count: placement has {placement.num_experts}, shape {shape.num_experts}")
    if placement.num_gpus != shape.num_gpus:
        out.append(f"gpu count: placement has {placement.num_gpus}, shape {shape.num_gpus}")
    for e, grp in enumerate(placement.edp_groups):
        if not grp:
            out.append(f"empty EDP group: expert {e}")
        if len(set(grp)) != len(grp):
            out.append(f"duplicate GPU: expert {e} group {grp}")
        out.extend(f"range: expert {e} references GPU {g} of {shape.num_gpus}"
                   for g in grp if not 0 <= g < shape.num_gpus)
    for g in range(min(placement.num_gpus, shape.num_gpus)):
        owner: dict[int, int] = {}
        for e in placement.hosted[g]:
            s = placement.slots[e]
            if s in owner:
                out.append(f"slot collision: experts {owner[s]} and {e} share slot {s} on GPU {g}")
            else:
                owner[s] = e
    if uniform:
        counts = placement.gpu_replica_counts()
        cap = sum(counts) // max(placement.num_gpus, 1)
        out.extend(f"uniformity: GPU {g} hosts {c} replicas, capacity {cap}" for g, c in enumerate(counts) if c != cap)
    return out


# ---------------------------------------------------------------------------
# Asymmetric placements (adaptive replacement, off the per-micro-batch path).
# Restated from placement.py:304-450 of the reference; the numpy generator is
# driven with the same calls in the same order, so a seed gives the reference's
# placement (pinned by tests/golden/sched_asym.json.gz).
# ---------------------------------------------------------------------------
_EXACT_GPU_CAP = 24


@dataclass(frozen=True)
class PlacementGraph:
    """Weighted hypergraph view of a placement: edge e = (sorted GPUs, weight)."""

    num_gpus: int
    edges: tuple

    @classmethod
    def from_placement(cls, placement: Placement, weights) -> "PlacementGraph":
        if len(weights) != placement.num_experts:
            raise DimensionError(f"{len(weights)} weights for {placement.num_experts} experts")
        out = []
        for grp, w in zip(placement.edp_groups, weights):
            w = Fraction(w)
            if w < 0:
                raise ContractViolation("edge weights must be >= 0")
            out.append((tuple(sorted(grp)), w))
        return cls(placement.num_gpus, tuple(out))


@dataclass(frozen=True)
class DensityReport:
    best_subset: tuple
    density: Fraction
    per_size: dict | None = None


def density_oracle(graph: PlacementGraph, mode: str = "exact", *, samples: int = 1000, seed: int = 0) -> DensityReport:
    """Maximum induced-subgraph density (= the min-max GPU load, Eq. 3)."""
    n = graph.num_gpus
    if mode == "exact":
        if n > _EXACT_GPU_CAP:
            raise CapacityError(f"exact density enumeration capped at {_EXACT_GPU_CAP} GPUs, got {n}")
        scale = math.lcm(*(w.denominator for _, w in graph.edges)) if graph.edges else 1
        ints = [int(w * scale) for _, w in graph.edges]
        if sum(ints) >= 1 << 62:
            raise CapacityError("edge weights too large for exact enumeration")
        W = np.zeros(1 << n, dtype=np.int64)
        for (gpus, _), wi in zip(graph.edges, ints):
            if wi and gpus:
                W[sum(1 << g for g in gpus)] += wi
        for b in range(n):  # subset-sum (zeta) transform
            v = W.reshape(-1, 2, 1 << b)
            v[:, 1, :] += v[:, 0, :]
        sizes = np.array([bin(S).count("1") for S in range(1 << n)])
        per_size, best, best_mask, best_k = {}, Fraction(0), 1, 1
        for k in range(1, n + 1):
            idx = np.flatnonzero(sizes == k)
            j = int(np.argmax(W[idx]))
            per_size[k] = Fraction(int(W[idx][j]), k * scale)
            if per_size[k] > best or (per_size[k] == best and k < best_k):
                best, best_mask, best_k = per_size[k], int(idx[j]), k
        return DensityReport(tuple(g for g in range(n) if best_mask >> g & 1), best, per_size)
    if mode == "sampled":
        rng = np.random.default_rng(seed)
        cands = [frozenset(range(n))] + [frozenset(g) for g, w in graph.edges if g and w > 0]
        for _ in range(samples):
            k = int(rng.integers(1, n + 1))
            cands.append(frozenset(int(g) for g in rng.choice(n, size=k, replace=False)))
        best, best_s = Fraction(0), frozenset([0])
        for S in cands:
            d = Fraction(sum(w for g, w in graph.edges if g and set(g) <= S), len(S))
            if d > best or (d == best and len(S) < len(best_s)):
                best, best_s = d, S
        return DensityReport(tuple(sorted(best_s)), best, None)
    raise ContractViolation(f"unknown density mode {mode!r}")


def _lowest_free_slots(num_gpus: int, groups) -> tuple:
    """Slot per expert: lowest index free on every GPU of its group."""
    used = [set() for _ in range(num_gpus)]
    out = []
    for grp in groups:
        taken = set().union(*(used[g] for g in grp)) if grp else set()
        s = 0
        while s in taken:
            s += 1
        out.append(s)
        for g in grp:
            used[g].add(s)
    return tuple(out)


def _draw_groups(rng, counts, capacities, retries: int = 64):
    """Random EDP groups with the given replica counts, GPUs drawn without
    replacement with probability proportional to their free capacity."""
    G = len(capacities)
    order = sorted(range(len(counts)), key=lambda e: (-counts[e], e))
    for _ in range(retries):
        free = list(capacities)
        groups = [None] * len(counts)
        ok = True
        for e in order:
            elig = [g for g in range(G) if free[g] > 0]
            if len(elig) < counts[e]:
                ok = False
                break
            w = np.array([free[g] for g in elig], dtype=np.float64)
            pick = rng.choice(len(elig), size=counts[e], replace=False, p=w / w.sum())
            grp = tuple(sorted(elig[int(i)] for i in pick))
            groups[e] = grp
            for g in grp:
                free[g] -= 1
        if ok:
            return groups
    return None


def random_placement(shape: ClusterShape, seed: int) -> Placement:
    """Uniform random d-subsets with balanced per-GPU replica counts."""
    if shape.d < 2:
        raise ConstructionError("random placement requires d >= 2")
    rng = np.random.default_rng(seed)
    base, rem = divmod(shape.num_experts * shape.d, shape.num_gpus)
    caps = [base] * shape.num_gpus
    for g in rng.permutation(shape.num_gpus)[:rem]:
        caps[int(g)] += 1
    groups = _draw_groups(rng, [shape.d] * shape.num_experts, caps)
    if groups is None:
        raise ConstructionError(f"could not sample a balanced placement for {shape} after bounded retries")
    return Placement(shape.num_gpus, tuple(groups), _lowest_free_slots(shape.num_gpus, groups))


def greedy_replica_counts(expert_loads, total_replica_slots: int, max_count: int | None = None) -> tuple:
    """One replica each, then every extra slot to the expert with the highest
    load per replica (ties -> lowest expert id), capped at max_count."""
    n = len(expert_loads)
    if total_replica_slots < n:
        raise ContractViolation(f"{total_replica_slots} slots cannot give {n} experts one replica each")
    if max_count is not None and max_count * n < total_replica_slots:
        raise ContractViolation("max_count too small to absorb all replica slots")
    counts = [1] * n
    heap = [(-Fraction(l), e) for e, l in enumerate(expert_loads)]
    heapq.heapify(heap)
    for _ in range(total_replica_slots - n):
        _, e = heapq.heappop(heap)
        counts[e] += 1
        if max_count is None or counts[e] < max_count:
            heapq.heappush(heap, (-Fraction(expert_loads[e], counts[e]), e))
    return tuple(counts)


def monte_carlo_placement(expert_loads, replica_counts, shape: ClusterShape, n_samples: int, seed: int) -> Placement:
    """Best of n_samples random layouts by maximum induced density."""
    counts = [int(c) for c in replica_counts]
    total = sum(counts)
    if total % shape.num_gpus:
        raise ContractViolation(f"replica counts sum to {total}, not a multiple of {shape.num_gpus} GPUs")
    if len(counts) != len(expert_loads):
        raise DimensionError("replica_counts and expert_loads disagree")
    for e, c in enumerate(counts):
        if not 1 <= c <= shape.num_gpus:
            raise ContractViolation(f"expert {e}: replica count {c} not in 1..{shape.num_gpus}")
    if n_samples < 1:
        raise ContractViolation("n_samples must be >= 1")
    caps = [total // shape.num_gpus] * shape.num_gpus
    rng = np.random.default_rng(seed)
    mode = "exact" if shape.num_gpus <= _EXACT_GPU_CAP else "sampled"
    best_groups, best_d = None, None
    for _ in range(n_samples):
        groups = _draw_groups(rng, counts, caps)
        if groups is None:
            raise ConstructionError("could not sample a placement honoring the replica counts")
        g = PlacementGraph(shape.num_gpus, tuple((tuple(sorted(x)), Fraction(w)) for x, w in zip(groups, expert_loads)))
        d = density_oracle(g, mode, samples=256, seed=seed).density
        if best_d is None or d < best_d:
            best_d, best_groups = d, groups
    return Placement(shape.num_gpus, tuple(best_groups), _lowest_free_slots(shape.num_gpus, best_groups))


def symmetric_placement(shape: ClusterShape, seed: int = 0, n_samples: int = 64) -> Placement:
    """Catalogued symmetric placement, else a Monte-Carlo / random fallback."""
    try:
        return cayley_symmetric(shape)
    except ConstructionError:
        if (shape.num_experts * shape.d) % shape.num_gpus == 0:
            return monte_carlo_placement([1] * shape.num_experts, [shape.d] * shape.num_experts, shape, n_samples, seed)
        return random_placement(shape, seed)
