"""Init-time placement constructors consumed by the MoE layer (host side).

Placements are built once, before training/serving, and uploaded to the
device scheduler; they are not on the per-micro-batch path.  Same names and
outputs as the reference (``/root/reference/pkg/src/harmonyep/placement.py``),
pinned by the reference's Cayley goldens (tests/golden/placements.json):

  cayley_symmetric      :207-265  catalogue: 8-cycle (p=3,q=1), 4x4 torus (4,2),
                                  K4,4 (3,2), complete graphs + XOR matchings (q >= p)
  identical_placement   :471-487  merged-EP layout (vanilla / merged_ep baselines)
  validate_placement    :490-528
"""

from __future__ import annotations

from .core import ClusterShape, ConstructionError, Placement

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
