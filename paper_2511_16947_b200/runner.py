"""The per-micro-batch caller of the layer, with real device work: the
reference's ``run_strategy`` harmony branch (``simulator.py:346-476``) driving
``MoELayer`` instead of its cost model.

Per micro-batch (``step``):
  * before it, every ``policy.check_interval`` micro-batches, the adaptive
    check (``simulator.py:379-392``): ``evaluate_and_maybe_replace`` on the
    moving-average ``LoadHistory`` (``adaptive.py:81-166``); a replacement
    swaps the layer's placement (``MoELayer.set_placement``; on a real EP
    group ``EPMoELayer.migrate`` moves the weights) and records the event;
  * the layer forward on the device (one stream, no host synchronisation);
  * a device-side record of the micro-batch — per-GPU loads, expert loads,
    all-to-all volumes, CUDA events around the forward — appended to a ring
    buffer (two small device copies), so the loop never waits on the GPU.

The host reads the ring only at an adaptive check (one sync every
``check_interval`` micro-batches, as the reference's policy runs there) and in
``metrics()``, which returns the reference's ``MicrobatchMetrics`` rows
(``simulator.py:121-131``) with ``layer_time`` = the MEASURED forward time in
µs; ``metrics_csv`` writes them under the reference's ``metrics.csv`` header
(``simulator.py:75-77``) so real runs can be diffed against simulated sweeps.
"""

from __future__ import annotations

import torch

from .adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace
from .core import ClusterShape, gpu_load_balance_ratio
from .sweep import METRICS_CSV_HEADER, MicrobatchMetrics


class LayerRunner:
    """Drive a single-device ``MoELayer`` (simulated EP group) micro-batch by
    micro-batch, with the reference's adaptive replacement policy and
    per-micro-batch metrics.  ``policy=None`` keeps the placement fixed."""

    def __init__(self, layer, policy: ReplacementPolicy | None = None, *, shape: ClusterShape | None = None,
                 seed: int = 0, capacity: int = 1024, stream=None):
        """shape: the ClusterShape the adaptive candidates are built for (default: d = the
        initial placement's replication, 2 if it is not uniform)."""
        self.layer = layer
        self.policy = policy
        self.seed = seed
        self.history = LoadHistory(policy.window) if policy is not None else None
        sizes = {len(g) for g in layer.placement.edp_groups}
        d = sizes.pop() if len(sizes) == 1 else 2
        self.shape = shape or ClusterShape(layer.G, layer.E, max(2, min(d, layer.G)))
        self.stream = stream
        self.capacity = capacity
        G, E = layer.G, layer.E
        # [gpu_load G | expert loads E | intra, inter, local]
        self._rec = torch.zeros(capacity, G + E + 3, dtype=torch.int64, device=layer.device)
        self._ev: list = [None] * capacity
        self.i = 0              # micro-batches issued
        self._pushed = 0        # micro-batches whose loads entered the history
        self.events: list[dict] = []
        self.last_decision = None
        self._checked_at = -1
        self.placements = [(0, layer.placement)]

    # ------------------------------------------------------------------
    def _record(self, b, st) -> None:
        layer, G, E = self.layer, self.layer.G, self.layer.E
        row = self._rec[self.i % self.capacity]
        tr = layer.sched.transfer
        with torch.cuda.stream(st):
            row[:G].copy_(layer.sched.gpu_load[:G])
            torch.sum(b.hist, dim=0, out=row[G:G + E])
            row[G + E:G + E + 2].copy_(tr[G * G + 7 * G:G * G + 7 * G + 2])  # intra, inter volume
            torch.sum(tr[G * G + 2 * G:G * G + 3 * G], dim=0, out=row[G + E + 2])  # local rows

    def _sync_history(self) -> None:
        """Host read of the records not yet in the history (one synchronisation)."""
        if self.history is None or self._pushed == self.i:
            return
        lo = max(self._pushed, self.i - self.capacity)
        rows = torch.stack([self._rec[j % self.capacity] for j in range(lo, self.i)]).cpu().tolist()
        G, E = self.layer.G, self.layer.E
        for r in rows[-self.history.capacity:]:
            self.history.push(r[G:G + E])
        self._pushed = self.i

    def _maybe_replace(self) -> None:
        p = self.policy
        if p is None or self.i == 0 or self.i % p.check_interval:
            return
        self._sync_history()
        if len(self.history) == 0:
            return
        if self._checked_at == self.i:
            return  # already decided at this index (check() then step())
        self._checked_at = self.i
        dec = evaluate_and_maybe_replace(self.layer.placement, self.history, p, self.shape, self.seed)
        self.last_decision = dec
        if dec.replaced:
            self.layer.set_placement(dec.placement)
            self.events.append(dec.to_event(self.i))
            self.placements.append((self.i, dec.placement))

    def check(self) -> None:
        """Run the adaptive check now if this micro-batch index is a check point (the
        check ``step`` runs before its forward), e.g. to settle the placement before a
        timed or graph-captured region."""
        self._maybe_replace()

    def step(self, x: torch.Tensor) -> torch.Tensor:
        """One micro-batch: adaptive check (every check_interval), forward, device record."""
        self._maybe_replace()
        st = self.stream if self.stream is not None else torch.cuda.current_stream()
        layer = self.layer
        b = layer.buffers(x.shape[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        layer.run(x, b, st)
        e1.record(st)
        self._record(b, st)
        self._ev[self.i % self.capacity] = (e0, e1)
        self.i += 1
        return b.out

    # ------------------------------------------------------------------
    def metrics(self) -> list[MicrobatchMetrics]:
        """The reference's per-micro-batch rows for the last ``capacity`` micro-batches,
        ``layer_time`` = measured forward time (µs, CUDA events on the launch stream)."""
        torch.cuda.synchronize(self.layer.device)
        G, E = self.layer.G, self.layer.E
        lo = max(0, self.i - self.capacity)
        rows = torch.stack([self._rec[j % self.capacity] for j in range(lo, self.i)]).cpu().tolist() if self.i else []
        out = []
        for j, r in zip(range(lo, self.i), rows):
            gl = r[:G]
            e0, e1 = self._ev[j % self.capacity]
            us = 1e3 * e0.elapsed_time(e1)
            out.append(MicrobatchMetrics(index=j, max_gpu_load=max(gl), balance_ratio=gpu_load_balance_ratio(gl),
                                         a2a_intra=r[G + E], a2a_inter=r[G + E + 1], local_volume=r[G + E + 2],
                                         layer_time=us, schedule_time_hidden=False,
                                         breakdown={"measured_us": us}))
        return out

    def metrics_csv(self, strategy: str = "harmony", s: float = 0.0, seed: int = 0) -> str:
        """``metrics.csv`` rows (reference header) with measured ``layer_time`` in µs."""
        lines = [METRICS_CSV_HEADER]
        for m in self.metrics():  # the reference's number formats (simulator.py:526-536)
            lines.append(f"{strategy},{s:.6f},{seed},{m.index},{m.max_gpu_load},{m.balance_ratio:.6f},{m.a2a_intra},"
                         f"{m.a2a_inter},{m.local_volume},{m.layer_time:.6f}")
        return "\n".join(lines) + "\n"
