"""Synthetic skewed workloads (benchmark input generator, host side).

``gen_zipf_workload`` reproduces the reference's counts-mode generator
(``/root/reference/pkg/src/harmonyep/simulator.py:157-195``): one random
popularity ranking per seed, then per source GPU a multinomial draw of
``tokens_per_gpu`` assignments.  Same numpy calls in the same order, so the
load matrices are identical to the reference's for a given numpy (pinned by
tests/golden/zipf_counts.json.gz).

``zipf_gate_bias`` turns the same ranking into a per-expert router bias for
token mode: selection scores ``logit + bias_e`` with
``bias_e = s * log p_e`` skew top-K picks toward popular experts while each
token still picks K distinct experts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ClusterShape, ContractViolation, LoadMatrix, TraceParseError


@dataclass(frozen=True)
class Workload:
    shape: ClusterShape
    micro_batches: tuple[LoadMatrix, ...]
    source: str = ""

    def __post_init__(self):
        for i, mb in enumerate(self.micro_batches):
            if (mb.num_experts, mb.num_gpus) != (self.shape.num_experts, self.shape.num_gpus):
                raise ContractViolation(
                    f"micro-batch {i} is {mb.num_experts}x{mb.num_gpus}, "
                    f"shape wants {self.shape.num_experts}x{self.shape.num_gpus}"
                )


def zipf_probabilities(num_experts: int, s: float) -> np.ndarray:
    w = np.arange(1, num_experts + 1, dtype=np.float64) ** (-float(s))
    return w / w.sum()


def zipf_expert_probs(num_experts: int, s: float, seed: int) -> tuple[np.ndarray, np.random.Generator]:
    rng = np.random.default_rng(seed)
    rank = rng.permutation(num_experts)
    p = np.empty(num_experts)
    p[rank] = zipf_probabilities(num_experts, s)
    return p, rng


def gen_zipf_workload(shape: ClusterShape, s: float, tokens_per_gpu: int, n_microbatches: int, seed: int) -> Workload:
    if s < 0:
        raise ContractViolation("zipf skew must be >= 0")
    if tokens_per_gpu < 0 or n_microbatches < 0:
        raise ContractViolation("token and micro-batch counts must be >= 0")
    p, rng = zipf_expert_probs(shape.num_experts, s, seed)
    mbs = []
    for _ in range(n_microbatches):
        m = np.zeros((shape.num_experts, shape.num_gpus), dtype=np.int64)
        for g in range(shape.num_gpus):
            m[:, g] = rng.multinomial(tokens_per_gpu, p)
        mbs.append(LoadMatrix.from_array(m))
    return Workload(shape, tuple(mbs), source=f"zipf(s={s}, seed={seed}, tokens_per_gpu={tokens_per_gpu})")


def zipf_gate_bias(num_experts: int, s: float, seed: int) -> np.ndarray:
    """Per-expert selection bias s*log(p_e) from the seeded Zipf ranking (fp32)."""
    p, _ = zipf_expert_probs(num_experts, s, seed)
    return (np.log(p) - np.log(p).mean()).astype(np.float32) if s > 0 else np.zeros(num_experts, np.float32)


def save_trace(workload: Workload, path: str) -> None:
    """Trace CSV ``microbatch,expert,gpu,tokens`` (non-zero entries), as the
    reference writes it (``simulator.py:196-203``)."""
    with open(path, "w", newline="") as f:
        f.write("microbatch,expert,gpu,tokens\n")
        for i, mb in enumerate(workload.micro_batches):
            for e, row in enumerate(mb.entries):
                for g, v in enumerate(row):
                    if v:
                        f.write(f"{i},{e},{g},{v}\n")


def load_trace(path: str, shape: ClusterShape) -> Workload:
    """Parse a trace CSV into a workload (``simulator.py:206-254``): header
    check, integer fields, range checks, repeated (mb, e, g) rows add up,
    missing micro-batches are all-zero.  Errors raise ``TraceParseError`` with
    the 1-based line number."""
    import csv
    import os

    if not os.path.exists(path):
        raise TraceParseError(f"no such trace file: {path}")
    per_mb: dict = {}
    with open(path, newline="") as f:
        reader = csv.reader(f)
        try:
            header = next(reader)
        except StopIteration:
            raise TraceParseError("empty file, expected a header row", 1) from None
        if [h.strip() for h in header] != ["microbatch", "expert", "gpu", "tokens"]:
            raise TraceParseError(f"bad header {header!r}, expected microbatch,expert,gpu,tokens", 1)
        for line_no, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != 4:
                raise TraceParseError(f"expected 4 fields, got {len(row)}", line_no)
            try:
                mb, e, g, v = (int(x) for x in row)
            except ValueError:
                raise TraceParseError(f"non-integer field in {row!r}", line_no) from None
            if mb < 0:
                raise TraceParseError(f"negative micro-batch index {mb}", line_no)
            if not (0 <= e < shape.num_experts):
                raise TraceParseError(f"expert {e} out of range 0..{shape.num_experts - 1}", line_no)
            if not (0 <= g < shape.num_gpus):
                raise TraceParseError(f"gpu {g} out of range 0..{shape.num_gpus - 1}", line_no)
            if v < 0:
                raise TraceParseError(f"negative token count {v}", line_no)
            m = per_mb.setdefault(mb, np.zeros((shape.num_experts, shape.num_gpus), dtype=np.int64))
            m[e, g] += v
    count = max(per_mb) + 1 if per_mb else 0
    mbs = [LoadMatrix.from_array(per_mb.get(i, np.zeros((shape.num_experts, shape.num_gpus), dtype=np.int64)))
           for i in range(count)]
    return Workload(shape, tuple(mbs), source=f"trace:{path}")
