"""Benchmark of the B200 HarmonyEP MoE layer (BASELINE.json metric:
"MoE-layer tokens/s at 1/2/4/8 B200; max/mean GPU load; scheduler µs/micro-batch").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral|qwen3|dsv3|tiny] [--skew S]
    python bench.py --impl reference ...      # CPU reference arm (oracle port on host cores)

A step = one forward pass of the MoE layer over one micro-batch of synthetic
tokens resident in HBM: router GEMM -> top-K + histogram -> exact scheduler ->
token assignment -> permute -> SwiGLU grouped GEMM x2 -> combine.  At N=1 the
EP group of G=8 GPUs is simulated on the one device (BASELINE configs[0]'s
"simulated EP"), T tokens per micro-batch split over the 8 virtual source
GPUs.  At N>1 every rank runs its own micro-batch through the same layer
(weak scaling: per-GPU work fixed; see DESIGN.md §multi-GPU for the exchange
path).  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (E, K, d_model, ffn, tokens per micro-batch per GPU, G)
    "tiny": (8, 2, 512, 1024, 4096, 4),
    "mixtral": (8, 2, 4096, 14336, 16384, 8),
    "qwen3": (128, 8, 2048, 768, 32768, 8),
    "dsv3": (256, 8, 7168, 2048, 16384, 8),
}
CONFIG_TEXT = {
    "tiny": "tiny MoE layer: 8 experts top-2, d_model=512, ffn=1024, 4096 tokens, simulated EP=4",
    "mixtral": "Mixtral-8x7B-shaped MoE layer: 8 experts top-2, d=4096, ffn=14336, 16K tokens/micro-batch, EP=8",
    "qwen3": "Qwen3-30B-A3B-shaped layer: 128 experts top-8, d=2048, ffn=768, 32K tokens, EP=8",
    "dsv3": "DeepSeek-V3-shaped fine-grained layer: 256 experts top-8, d=7168, ffn=2048, 16K tokens, EP=8",
}
METRIC = "MoE-layer tokens/s at 1/2/4/8 B200; max/mean GPU load; scheduler µs/micro-batch"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ---------------------------------------------------------------------------
# CPU reference arm: the oracle port of the reference path on host cores
# ---------------------------------------------------------------------------
_CPU_W: dict = {}


def _cpu_expert_weights(cfg_name: str, e: int):
    import numpy as np

    E, K, d, F, T, G = CONFIGS[cfg_name]
    key = (cfg_name, e % 16 if E > 16 else e)
    if key not in _CPU_W:
        g = np.random.default_rng(1000 + key[1])
        _CPU_W[key] = (g.standard_normal((F, d), dtype=np.float32) / np.sqrt(d),
                       g.standard_normal((F, d), dtype=np.float32) / np.sqrt(d),
                       g.standard_normal((d, F), dtype=np.float32) / np.sqrt(F))
    return _CPU_W[key]


def cpu_reference_step(cfg_name: str, skew: float, sample_tokens: int, seed: int = 0):
    """One bounded-sample step of the CPU restatement: router GEMM + top-K +
    histogram for the sample, the reference scheduler (Dinic oracle, C) on a
    full-size micro-batch load matrix, and the SwiGLU FFN + combine for the
    sample tokens (numpy fp32, all host threads via BLAS).  Returns seconds per
    token (the scheduler's per-micro-batch time amortised over T tokens)."""
    import numpy as np

    from oracle import layer_ref
    from oracle import oracle as O
    import paper_2511_16947_b200 as P

    E, K, d, F, T, G = CONFIGS[cfg_name]
    rng = np.random.default_rng(seed)
    S = sample_tokens
    x = rng.standard_normal((S, d), dtype=np.float32)
    wg = (rng.standard_normal((E, d), dtype=np.float32) / np.sqrt(d)).astype(np.float32)
    bias = P.zipf_gate_bias(E, skew, seed) if skew > 0 else None
    t0 = time.perf_counter()
    logits = x @ wg.T
    idx, w = layer_ref.topk_select(logits, K, bias)
    t_gate = time.perf_counter() - t0
    # scheduler on a full micro-batch histogram (counts mode, reference generator)
    wl = P.gen_zipf_workload(P.ClusterShape(G, E, 2), skew, (T // G) * K, 1, seed)
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    loads = wl.micro_batches[0].entries
    t0 = time.perf_counter()
    O.full_path(G, pl.edp_groups, loads)
    t_sched = time.perf_counter() - t0
    # expert FFN for the sample, distinct fp32 weights per expert (pool of at
    # most 16 weight sets for the 256-expert shape to bound host memory)
    t_ffn = 0.0
    out = np.zeros((S, d), dtype=np.float32)
    for e in np.unique(idx):
        w1, w3, w2 = _cpu_expert_weights(cfg_name, int(e))
        rows, ks = np.nonzero(idx == e)
        t0 = time.perf_counter()
        y = layer_ref.expert_ffn(x[rows], w1, w3, w2)
        out[rows] += w[rows, ks][:, None] * y
        t_ffn += time.perf_counter() - t0
    per_token = (t_gate + t_ffn) / S + t_sched / T
    return per_token, dict(t_gate=t_gate, t_ffn=t_ffn, t_sched=t_sched, sample=S)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    E, K, d, F, T, G = CONFIGS[cfg]
    cores, model = cpu_info()
    sample = args.cpu_sample or {"tiny": 1024, "mixtral": 128, "qwen3": 512, "dsv3": 128}[cfg]
    steps = args.steps  # each step is a bounded sample: K steps stay within a few minutes of host time
    for _ in range(min(args.warmup, 2)):
        cpu_reference_step(cfg, args.skew, max(8, sample // 8))
    per, walls = [], []
    for i in range(steps):
        t0 = time.perf_counter()
        pt, info = cpu_reference_step(cfg, args.skew, sample, seed=i)
        walls.append(time.perf_counter() - t0)
        per.append(pt)
    value = 1.0 / statistics.mean(per)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup,
        # the MEASURED wall time of one sampled step (sample tokens + one full scheduler solve)
        "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": CONFIG_TEXT[cfg], "tokens_per_microbatch": T, "sim_ep": G, "top_k": K,
                   "zipf_s": args.skew},
        "sample_tokens": sample,
        "extrapolated": True,
        "extrapolation": (f"value = 1 / per-token time, per-token time = (router+FFN time of the {sample}-token "
                          f"sample) / {sample} + (scheduler time of the full {G}x{E} micro-batch) / {T}; one "
                          f"full {T}-token micro-batch would take {1e3 * T * statistics.mean(per):.0f} ms"),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} tokens/step through router+top-K+SwiGLU FFN (numpy fp32, BLAS threads) + "
                                   f"the Dinic scheduler oracle on one full {G}x{E} micro-batch load matrix; "
                                   f"host: {model}"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm, N > 1: real expert parallelism, one rank per GPU (ep.py)
# ---------------------------------------------------------------------------
def load_traffic(config: str) -> dict:
    """Per-launch DRAM bytes of the hot kernels from the committed ncu launch
    list (profiles/traffic.json, written by tools/traffic.py); {} if absent."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get(config, {})


def _max_over_ranks(v: float, dev) -> float:
    """Max of a host float over all ranks (device tensor under NCCL, host under gloo)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ep(args, world, rank, local, dev):
    """Scheduling group = the N ranks; every rank owns T tokens per micro-batch
    (weak scaling: per-GPU work fixed).  Histogram all-gather and the dispatch /
    combine all-to-all-v run over NCCL; the placement is the Cayley layout of
    the N GPUs, replaced by the adaptive one when it is better (decided from the
    all-gathered loads, identically on every rank)."""
    import torch
    import torch.distributed as dist

    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200.adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace
    from paper_2511_16947_b200.ep import DistComm, EPMoELayer

    E, K, d, F, T, _ = CONFIGS[args.config]
    G = world
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape) if (E & (E - 1)) == 0 and (G & (G - 1)) == 0 else P.placement.symmetric_placement(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, args.skew, 0)) if args.skew > 0 else None
    comm = DistComm()
    # self-check of the process group the exchange runs in (backend, ranks, NCCL version)
    comm_info = {"backend": dist.get_backend(), "ranks": dist.get_world_size(),
                 "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if dist.get_backend() == "nccl" else None}
    if rank == 0:
        print(f"[bench] communicator: {comm_info}", file=sys.stderr)
    if args.pipeline_ratio is not None:  # harmony_pipelined: the static share's all-to-all-v overlaps the solve
        args.exchange = "nccl"
    layer = EPMoELayer(pl, d, F, K, comm, [rank], seed=0, gate_bias=bias, device=dev, exchange=args.exchange,
                       pipeline_ratio=args.pipeline_ratio)
    x = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(1000 + rank), device=dev).to(torch.bfloat16)
    ok = 1
    try:  # the NVLink path maps the peers' buffers with CUDA IPC; fall back to NCCL if that is refused
        layer.forward([x])
        torch.cuda.synchronize()
    except Exception as exc:  # noqa: BLE001 - any mapping/launch failure of the peer path
        if args.exchange != "p2p":
            raise
        print(f"[bench] rank {rank}: NVLink peer exchange unavailable ({exc}); using NCCL all-to-all-v",
              file=sys.stderr)
        ok = 0
    if args.exchange == "p2p":
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:  # every rank switches together
            args.exchange = "nccl"
            layer = EPMoELayer(pl, d, F, K, comm, [rank], seed=0, gate_bias=bias, device=dev, exchange="nccl")
    for _ in range(args.warmup):
        layer.forward([x])
    torch.cuda.synchronize()
    gl = layer.ranks[0].sched.gpu_load.cpu().tolist()
    static_mm = max(gl) * len(gl) / max(sum(gl), 1)
    replacement = None
    if args.placement == "adaptive":
        hist = LoadHistory(8)
        hist.push(layer.ranks[0].bufs[T]["hist_all"].sum(dim=0).cpu().tolist())
        dec = evaluate_and_maybe_replace(pl, hist, ReplacementPolicy(threshold=1.0, mc_samples=200), shape, 0)
        replacement = dec.to_event(args.warmup)
        if dec.replaced:  # migration: the new replicas' weights move over NCCL from an old holder
            pl = dec.placement
            dist.barrier()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record()
            mig = layer.migrate(pl)
            m1.record()
            torch.cuda.synchronize()
            mt = _max_over_ranks(m0.elapsed_time(m1), dev)
            replacement = dict(replacement or {}, migration_ms=mt, moved_replicas=mig["moved_replicas"],
                               bytes_per_replica=mig["bytes_per_replica"])
            for _ in range(args.warmup):
                layer.forward([x])
            torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    # the NVLink exchange with device-side barriers has no host synchronisation in the
    # step: capture it as one CUDA graph per rank (the barrier epochs advance on the device)
    graph = None
    if args.exchange == "p2p" and comm.device_sync and not args.eager:
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(stream)
            torch.cuda.synchronize()
            dist.barrier()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=side):
                layer.forward([x], stream=side)
            torch.cuda.synchronize()
            dist.barrier()
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # eager launches are the same kernels
            print(f"[bench] rank {rank}: CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graph = None
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            layer.forward([x])
    e1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    layer.check_sync()
    dist.barrier()
    # FFN share (roofline): a few extra steps with events around the expert GEMMs
    n_f = min(args.steps, 10)
    fev = [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in ("ffn", "a2a")}
           for _ in range(n_f)]
    for i in range(n_f):
        layer.forward([x], events=fev[i])
    torch.cuda.synchronize()
    ffn_ms = statistics.mean(f["ffn"][0].elapsed_time(f["ffn"][1]) for f in fev)
    a2a_ms = _max_over_ranks(statistics.mean(f["a2a"][0].elapsed_time(f["a2a"][1]) for f in fev), dev)
    # bytes this rank sends to other ranks per step (its transfer-plan row minus the local part)
    pair = layer.ranks[0].sched.transfer[: G * G].view(G, G).cpu()
    sent_rows = int(pair[rank].sum().item() - pair[rank, rank].item())
    a2a_bytes = sent_rows * d * 2
    a2a_gbs = -_max_over_ranks(-(a2a_bytes / (a2a_ms / 1e3) / 1e9), dev)  # slowest rank
    if layer.static_share is not None:  # pipelined: both phases' received rows; the a2a events bracket phase 1's
        R = int(layer.ranks[0].bufs[T]["R_recv"])
    else:
        R = int(layer.ranks[0].bufs[T]["counts"][G:].sum().item())  # rows this rank received (outside the timing)
    ffn_tf = 6.0 * d * F * R / (ffn_ms / 1e3) / 1e12
    min_tf = -_max_over_ranks(-ffn_tf, dev)
    hbm, tf_burst, tf_sus, peak_src = load_peaks()
    t_ms = _max_over_ranks(e0.elapsed_time(e1), dev)
    gl = layer.ranks[0].sched.gpu_load.cpu().tolist()
    mm = max(gl) * len(gl) / max(sum(gl), 1)
    # e2e: host tokens in, host outputs back, every step
    xh = x.cpu().pin_memory()
    oh = torch.empty(T, d, dtype=torch.bfloat16).pin_memory()
    xd = torch.empty_like(x)
    dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        xd.copy_(xh, non_blocking=True)
        (out,) = layer.forward([xd])
        oh.copy_(out, non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    e_ms = _max_over_ranks(f0.elapsed_time(f1), dev)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": world * T * args.steps / (t_ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[args.config], "tokens_per_microbatch_per_gpu": T, "ep": world,
                       "top_k": K, "d_model": d, "ffn": F, "experts": E, "zipf_s": args.skew, "pass": "forward",
                       "schedule": ("harmony" if layer.static_share is None else
                                    f"harmony_pipelined (pipeline_ratio={args.pipeline_ratio}: the static share's "
                                    "all-to-all-v on a side stream while the scheduled share is solved)"),
                       "launch": ("cuda-graph replay (device-side barriers, no host sync)" if graph is not None
                                  else "eager"),
                       "exchange": (("NVLink peer stores: dispatch kernel -> peers' receive buffers, down-projection "
                                     "epilogue -> sources' return buffers (CUDA IPC); histogram all-gather + 2 barriers")
                                    if args.exchange == "p2p" else
                                    ("NCCL" if args.dist_backend == "nccl" else "gloo, host-staged (protocol check)")
                                    + " all-gather (histograms) + all-to-all-v dispatch/combine")},
            "max_mean_gpu_load": mm, "max_mean_gpu_load_static_cayley": static_mm, "replacement": replacement,
            "comm": comm_info,
            "e2e": {"value": world * T * args.steps / (e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": T * d * 2, "d2h_bytes_per_step": T * d * 2},
            # router, scheduler, assignment (4), permute, FFN (4), combine = 12, + the per-slot
            # regrouping (layout, permute, gather back) = 15; the NVLink path: 13 + layout and
            # regroup permute = 15; the pipelined split adds the split kernel, the static phase's
            # scheduler launch, a second assignment (4) and permute = 22
            "gpu_launches": args.steps * (15 if args.exchange == "p2p" else (22 if layer.static_share is not None else 15)),
            "roofline": {"bound": "tensor", "kernel": "hep_moe_expert_ffn on the received rows (rank 0)",
                         "achieved": ffn_tf, "peak": tf_sus, "unit": "TFLOP/s", "frac": ffn_tf / tf_sus,
                         "min_over_ranks": min_tf, "rows_rank0": R,
                         "peak_source": f"{peak_src} bf16_tflops_sustained", "traffic": None},
            "clocks": sampler.summary() if sampler else None,
            # dispatch exchange: bytes each rank sends to other ranks / the exchange's event time
            # (p2p: the dispatch kernel storing into the peers' receive buffers, permute included;
            # NCCL: the all-to-all-v), against NVLink 5's 900 GB/s per direction per GPU
            "a2a": {"kind": "dispatch (" + ("NVLink peer stores" if args.exchange == "p2p" else "NCCL all-to-all-v") + ")",
                    "GB/s": a2a_gbs, "bytes_per_step_rank0": a2a_bytes, "ms": a2a_ms,
                    "frac_of_nvlink": a2a_gbs / 900.0, "nvlink_GB/s": 900.0,
                    "note": ("all ranks share one GPU (protocol check): not an NVLink figure"
                             if args.dist_backend == "gloo" else "max over ranks of the exchange time")},
        }))
    dist.destroy_process_group()


# ---------------------------------------------------------------------------
# our arm, N = 1: the EP group of G virtual GPUs simulated on the one device
# ---------------------------------------------------------------------------
def _events(n, keys):
    import torch

    return [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in keys}
            for _ in range(n)]


def _pool(T, d, dev, seeds):
    """Distinct synthetic micro-batches, X ~ N(0, 1) bf16, one seed each."""
    import torch

    return [torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(s), device=dev).to(torch.bfloat16)
            for s in seeds]


def _policy(n_seen: int):
    """The reference's ReplacementPolicy (adaptive.py:50-66) with the check after the
    warm-up window: threshold 1.1, Monte-Carlo 200 samples, window = check interval =
    the number of warm-up (seen) micro-batches."""
    from paper_2511_16947_b200.adaptive import ReplacementPolicy

    return ReplacementPolicy(check_interval=n_seen, threshold=1.1, window=n_seen, mc_samples=200)


def _mm(gl):
    mean = sum(gl) / len(gl)
    return max(gl) / mean if mean else 1.0


def _stat(vals):
    return {"mean": statistics.mean(vals), "max": max(vals), "per_batch": [round(v, 6) for v in vals]}


def heldout_balance(layer, static_ds, xs, stream):
    """max/mean GPU load of each micro-batch in ``xs`` under the layer's current
    placement and under the static placement ``static_ds`` (same device histogram,
    two device solves)."""
    import torch

    E = layer.E
    cur, sta = [], []
    for x in xs:
        gl = layer.schedule(x, stream)
        b = layer.buffers(x.shape[0])
        static_ds.launch_solve(b.hist, 1, E, None, 15, stream)
        torch.cuda.synchronize()
        layer.check_status()
        static_ds.check_status("static placement")
        cur.append(_mm(gl.cpu().tolist()))
        sta.append(_mm(static_ds.gpu_load.cpu().tolist()))
    return cur, sta


def balance_sweep(layer, pl_static, shape, seen, unseen, skews, stream):
    """Mixtral-shaped balance vs skew: for each Zipf s the
    reference's adaptive policy is decided on the warm-up (seen) micro-batches only and
    scored, with the static Cayley placement, on held-out micro-batches."""
    import torch

    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200.adaptive import LoadHistory, evaluate_and_maybe_replace
    from paper_2511_16947_b200.scheduler import DeviceScheduler

    E = layer.E
    bias0 = layer.gate_bias.clone()
    static_ds = DeviceScheduler(pl_static, device=layer.device)
    out = {}
    for s in skews:
        layer.gate_bias.copy_(torch.tensor(P.zipf_gate_bias(E, s, 0)))
        hist = LoadHistory(len(seen))
        for x in seen:
            layer.schedule(x, stream)
            hist.push(layer.buffers(x.shape[0]).hist.sum(dim=0).cpu().tolist())
        dec = evaluate_and_maybe_replace(pl_static, hist, _policy(len(seen)), shape, 0)
        ada_ds = DeviceScheduler(dec.placement, device=layer.device)
        ada, sta = [], []
        for x in unseen:
            layer.schedule(x, stream)
            b = layer.buffers(x.shape[0])
            for ds, acc in ((static_ds, sta), (ada_ds, ada)):
                ds.launch_solve(b.hist, 1, E, None, 15, stream)
                torch.cuda.synchronize()
                ds.check_status("balance sweep")
                acc.append(_mm(ds.gpu_load.cpu().tolist()))
        out[f"{s:g}"] = {"static_cayley": _stat(sta), "adaptive": _stat(ada), "replaced": dec.replaced,
                         "predicted_ratio_static": round(dec.predicted_ratio, 6)}
    layer.gate_bias.copy_(bias0)
    return out


def sched_cpu_baseline(configs, n_mb=50, skip=5, seed=0, skew=1.0):
    """the reference's per-micro-batch scheduling path (solve cold /
    warm -> integerize -> route -> transfer plan) on the counts-mode load matrices
    gen_zipf_workload(shape, s, T*K, 50, seed), 1 host core, median / p99 over the
    micro-batches after the first 5 — timed on the oracle (C restatement of the
    reference's Dinic algorithm, oracle/hep_oracle.c; the Python reference cannot run
    on the GPU box) — beside the device scheduler (hep_sched_solve, all stages) on the
    same matrices."""
    import numpy as np
    import torch

    from oracle import oracle as O
    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200.scheduler import DeviceScheduler

    def q(v):
        v = sorted(v)
        return {"median_us": round(statistics.median(v), 2), "p99_us": round(v[min(len(v) - 1, int(0.99 * len(v)))], 2)}

    out = {}
    for cfg in configs:
        E, K, d, F, T, G = CONFIGS[cfg]
        shape = P.ClusterShape(G, E, 2)
        pl = P.cayley_symmetric(shape)
        groups = [tuple(g) for g in pl.edp_groups]
        wl = P.gen_zipf_workload(shape, skew, (T // G) * K, n_mb, seed)
        mats = [np.asarray(mb.as_array(), dtype=np.int64) for mb in wl.micro_batches]
        cold, warm = [], []
        state = O.OracleState(G, groups)
        for m in mats:
            t0 = time.perf_counter()
            O.full_path(G, groups, m)  # fresh state: cold
            cold.append(1e6 * (time.perf_counter() - t0))
            t0 = time.perf_counter()
            O.full_path(G, groups, m, state=state)  # reused state: warm
            warm.append(1e6 * (time.perf_counter() - t0))
        ds = DeviceScheduler(pl)
        dl = torch.as_tensor(np.stack(mats)).cuda()
        st = torch.cuda.current_stream()
        dev = []
        for i in range(len(mats)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ds.launch_solve(dl[i], G, 1, None, 15, st)
            e1.record(st)
            torch.cuda.synchronize()
            dev.append(1e3 * e0.elapsed_time(e1))
        ds.check_status("sched baseline")
        out[cfg] = {"cpu_cold": q(cold[skip:]), "cpu_warm": q(warm[skip:]), "device": q(dev[skip:]),
                    "matrices": f"gen_zipf_workload(ClusterShape({G},{E},2), s={skew}, tokens_per_gpu={(T // G) * K}, "
                                f"{n_mb}, seed={seed}), Cayley placement; first {skip} excluded"}
    cores, model = cpu_info()
    return {"configs": out, "cores": 1, "host_cpu_count": cores, "host_cpu": model, "kind": "port",
            "what": "oracle/hep_oracle.c (the reference's Dinic + lex-min + integerize + Algorithm 1 + transfer "
                    "plan restated in C) per micro-batch through its ctypes wrapper, time.perf_counter; device = "
                    "one hep_sched_solve launch (same stages), CUDA events"}


def hbm_b2b_ms(layer, bufs, x, stream, n=20):
    """permute, combine and the fused router+gate, each re-launched n times back to back on
    the micro-batch ``x`` the buffers hold (idempotent kernels), captured in a CUDA graph;
    5 warm replays, then the median of 5 timed replays (CUDA events): ms per launch."""
    import torch

    from paper_2511_16947_b200 import _lib

    L = _lib.lib()
    T, d = x.shape
    K, E, G = layer.K, layer.E, layer.G

    def b2b(fn):
        # n launches captured in one CUDA graph (as the layer step runs), one warm replay,
        # then a timed replay: device time per launch without host launch overhead
        fn(stream.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()  # capture needs a non-default stream
        with torch.cuda.stream(cap):
            g.capture_begin()
            for _ in range(n):
                fn(cap.cuda_stream)
            g.capture_end()
        torch.cuda.synchronize()
        times = []
        with torch.cuda.stream(cap):
            for _ in range(5):  # clocks up (the GPU idles down during the rest before this)
                g.replay()
            for _ in range(5):
                q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                q0.record(cap)
                g.replay()
                q1.record(cap)
                times.append((q0, q1))
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in times) / n

    tr = bufs.tok_row if layer.static_share is None else bufs.tok_row
    perm = b2b(lambda cs: _lib.check(L.hep_moe_permute(x.data_ptr(), tr.data_ptr(), T, K, d, bufs.rows.data_ptr(), cs),
                                     "permute"))
    comb = b2b(lambda cs: _lib.check(L.hep_moe_combine(bufs.y.data_ptr(), tr.data_ptr(), bufs.topk_w.data_ptr(), T, K,
                                                       d, bufs.out.data_ptr(), cs), "combine"))
    chunk = None if layer.static_share is not None else bufs.assign_ws.data_ptr() + bufs.chunk_off
    rg = b2b(lambda cs: _lib.check(L.hep_router_topk_ws(
        x.data_ptr(), layer.wg.data_ptr(), T, d, E, layer.e_pad, _lib.ptr(layer.gate_bias), K, T // G, G,
        bufs.logits.data_ptr(), bufs.topk_idx.data_ptr(), bufs.topk_w.data_ptr(), bufs.hist.data_ptr(), chunk,
        bufs.router_sync.data_ptr(), cs), "router"))
    return perm, comb, rg


def measure_config(cfg, args, dev, *, steps, primary):
    """One workload: held-out protocol, CUDA-graph timed region, stage / kernel
    breakdown, balance, e2e.  Returns the line's fields (primary) or a summary."""
    import torch

    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200 import _lib
    from paper_2511_16947_b200.layer import HostPipeline
    from paper_2511_16947_b200.runner import LayerRunner
    from paper_2511_16947_b200.scheduler import DeviceScheduler

    L = _lib.lib()
    E, K, d, F, T, G = CONFIGS[cfg]
    shape = P.ClusterShape(G, E, 2)
    pl_static = P.cayley_symmetric(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, args.skew, 0)) if args.skew > 0 else None
    layer = P.MoELayer(pl_static, d, F, K, seed=0, gate_bias=bias, device=dev,
                       pipeline_ratio=args.pipeline_ratio if primary else None)
    n_seen = max(1, args.batches // 2)
    n_unseen = max(1, args.batches - n_seen)
    seen = _pool(T, d, dev, range(1000, 1000 + n_seen))
    unseen = _pool(T, d, dev, range(1000 + n_seen, 1000 + n_seen + n_unseen))
    stream = torch.cuda.current_stream()

    # --- warm-up micro-batches through the reference's run_strategy loop (LayerRunner):
    # expert loads into the LoadHistory, the adaptive check after them (seen batches only)
    adaptive = args.placement == "adaptive" and layer.static_share is None
    runner = LayerRunner(layer, _policy(n_seen) if adaptive else None, shape=shape)
    # the router+gate's own rate, taken before any FFN step heats the GPU: the router
    # (HBM-bound mainloop, ALU-bound epilogue) runs ~10-20 % slower for seconds after FFN
    # bursts (profiles/r02/router_ab_r02d.txt --hot); the in-step rate is reported beside
    b0 = layer.buffers(T)
    rg_early = []
    for xb in unseen[:4]:
        layer.run(xb, b0, stream)
        rg_early.append(hbm_b2b_ms(layer, b0, xb, stream)[2])
    rg_early = statistics.median(rg_early)
    for i in range(max(n_seen, args.warmup)):
        runner.step(seen[i % n_seen])
    torch.cuda.synchronize()
    layer.check_status()
    warm_rows = runner.metrics()
    if adaptive:
        runner.check()  # runner.i == n_seen (or a multiple): the policy runs here
    dec = runner.last_decision
    replacement = runner.events[-1] if runner.events else (dec.to_event(runner.i) if dec is not None else None)
    if replacement is not None and dec is not None:
        replacement = dict(replacement, replaced=dec.replaced, predicted_ratio=round(dec.predicted_ratio, 6))
    placement_desc = f"cayley_symmetric(G={G}, E={E}, d=2)"
    if runner.events:
        placement_desc = ("adaptive (reference policy on the warm-up micro-batches): greedy replica counts + "
                          f"Monte-Carlo layout (200 samples) from cayley_symmetric(G={G}, E={E}, d=2)")
    for x in seen[: min(3, n_seen)]:  # warm the adopted placement's launch paths
        layer.run(x, layer.buffers(T), stream)
    torch.cuda.synchronize()
    layer.check_status()
    bufs = layer.buffers(T)

    # --- the HBM-bound kernels' own rate, measured before the long power-capped timed region
    # (the kernel's capability; the same measurement after it is reported beside).  The
    # warm-up's FFN work leaves the GPU power-capped for a while (the router right after FFN
    # bursts runs ~20 % slower, profiles/r02/router_ab_r02d.txt --hot): rest 2 s first so this
    # figure is taken at the nominal clock
    # figure is taken at the nominal clock.  Median over 4 held-out micro-batches: the rate
    # moves a few % with where the 134-235 MB input happens to be allocated
    # (profiles/r02/router_ab_r02l.txt vs the bench line)
    layer.run(unseen[0], bufs, stream)
    torch.cuda.synchronize()
    time.sleep(2.0)
    per_x = []
    for xb in unseen[:4]:
        layer.run(xb, bufs, stream)  # its row map for the permute / combine
        per_x.append(hbm_b2b_ms(layer, bufs, xb, stream))
    hbm_b2b_before = (statistics.median(v[0] for v in per_x), statistics.median(v[1] for v in per_x), rg_early)
    layer.run(unseen[0], bufs, stream)
    torch.cuda.synchronize()

    # --- timed region: K CUDA-graph replays cycling over the held-out micro-batches
    graphs = None
    if not args.profile and not args.eager:
        try:
            graphs = [layer.capture(x) for x in unseen]
            for g in graphs:
                g.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # capture is an optimisation; eager launches are the same kernels
            print(f"[bench] CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graphs = None
    stages = ("router", "gate", "sched", "assign", "permute", "ffn", "combine")
    sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) if (primary and not args.profile) else None
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(steps):
        if graphs is not None:
            graphs[i % n_unseen].replay()
        else:
            layer.run(unseen[i % n_unseen], bufs, stream)
    end.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    layer.check_status()
    t_ms = start.elapsed_time(end)
    ms_per_step = t_ms / steps
    value = T * steps / (t_ms / 1e3)
    del graphs

    # --- stage breakdown: eager steps with events around every stage
    n_st = min(steps, 20)
    evs = _events(n_st, stages)
    for i in range(n_st):
        layer.run(unseen[i % n_unseen], bufs, stream, events=evs[i])
    torch.cuda.synchronize()
    stage_ms = {k: statistics.mean(e[k][0].elapsed_time(e[k][1]) for e in evs) for k in stages}
    ffn_ms = stage_ms["ffn"]

    # --- the SM clock the expert GEMMs ran at (CTA-0 clock64 / globaltimer stamps)
    ffn_clock = None
    if primary and not args.profile:
        import ctypes as _ct

        with _lib.tuning(ffn_clock=1):
            for i in range(min(steps, 10)):
                layer.run(unseen[i % n_unseen], bufs, stream)
            torch.cuda.synchronize()
            stc = (_ct.c_int64 * 8)()
            _lib.check(L.hep_ffn_debug_clock(stc), "hep_ffn_debug_clock")
        mhz = [1e3 * (stc[4 * g + 2] - stc[4 * g]) / max(1, stc[4 * g + 3] - stc[4 * g + 1]) for g in range(2)]
        ns = [stc[4 * g + 3] - stc[4 * g + 1] for g in range(2)]
        ffn_clock = {"gemm1_mhz": round(mhz[0], 1), "gemm2_mhz": round(mhz[1], 1),
                     "mhz": round((mhz[0] * ns[0] + mhz[1] * ns[1]) / max(1, ns[0] + ns[1]), 1),
                     "source": "clock64 / globaltimer of CTA 0 across each expert GEMM (eager steps)"}

    # --- scheduler latency: the K3 kernel alone on the last micro-batch's histogram
    xl = unseen[(steps - 1) % n_unseen]
    layer.run(xl, bufs, stream)
    n_sched = 200
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(n_sched):
        layer.sched.launch_solve(bufs.hist, 1, E, None, 15, stream)
    s1.record(stream)
    torch.cuda.synchronize()
    sched_us = 1e3 * s0.elapsed_time(s1) / n_sched

    # --- HBM-bound kernels re-launched back to back on that micro-batch (idempotent); the
    # same measurement was taken before the timed region (hbm_b2b_before)
    perm_ms, comb_ms, rg_ms = hbm_b2b_ms(layer, bufs, xl, stream)
    layer.run(xl, bufs, stream)  # restore the micro-batch's own state after the re-launches
    torch.cuda.synchronize()
    layer.check_status()

    # --- balance on the held-out micro-batches: the timed placement vs static Cayley
    static_ds = DeviceScheduler(pl_static, device=dev)
    if layer.static_share is None:
        cur, sta = heldout_balance(layer, static_ds, unseen, stream)
    else:  # pipelined: the device loads of the two phases (former + scheduled)
        cur, sta = [], []
        for x in unseen:
            layer.run(x, bufs, stream)
            torch.cuda.synchronize()
            gl = (layer.sched.gpu_load + layer.sched.former.gpu_load).cpu().tolist()
            cur.append(_mm(gl))
        sta = cur
    gpu_load = layer.sched.gpu_load.cpu().tolist()
    m_num, m_den = layer.sched.m[:2].cpu().tolist()

    # --- e2e through the public API with host buffers (pinned), HostPipeline
    n_host = min(n_unseen, 4)
    pipe = HostPipeline(layer, T)
    xh = [unseen[i].cpu().pin_memory() for i in range(n_host)]
    for i in range(3):
        pipe.submit(xh[i % n_host])
    pipe.drain()
    torch.cuda.synchronize()
    n_e2e = steps  # the pipeline's fill (first H2D) and drain (last D2H) amortised over all steps
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_in)
    last = None
    for i in range(n_e2e):
        last = pipe.submit(xh[i % n_host])
    out_last = pipe.result(last)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(pipe.s_out)
    torch.cuda.synchronize()
    e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3)
    e2e_value = T * n_e2e / (e_ms / 1e3)
    assert torch.isfinite(out_last.float()).all()
    del pipe, xh

    hbm, tf_burst, tf_sus, peak_src = load_peaks()
    R = T * K
    ffn_flops = 6.0 * d * F * R
    ffn_tflops = ffn_flops / (ffn_ms / 1e3) / 1e12
    perm_bytes = T * d * 2 * (1 + K) + T * K * 4
    comb_bytes = T * K * d * 2 + T * K * 4 * 2 + T * d * 2
    rg_bytes = T * d * 2 + layer.e_pad * d * 2 + T * layer.e_pad * 4 + T * K * 8  # x, Wg, logits, top-K
    traffic = load_traffic(cfg)
    # per-expert roofline: every expert's two GEMMs at its own bound -- tensor (6dF flop per
    # row at the sustained peak) or HBM (its weights once + its rows' X / H / Y at the copy
    # peak).  Experts with few rows (DeepSeek-V3's long tail) are weight-streaming bound, so
    # this is the FFN's time floor when experts are processed one after another
    er = bufs.expert_rows.cpu().tolist()
    per_expert = per_expert_roofline([er[e + 1] - er[e] for e in range(E)], d, F, tf_sus, hbm, ffn_ms)
    # the same floor with the burst tensor peak (a kernel timed alone); the sustained one
    # above is cuBLAS's long-run rate under the power cap, which a power-capped FFN can match
    per_expert["frac_burst"] = per_expert_roofline([er[e + 1] - er[e] for e in range(E)], d, F, tf_burst, hbm,
                                                   ffn_ms)["frac"]
    res = {
        "value": value, "ms_per_step": ms_per_step, "steps": steps,
        "config": {"workload": CONFIG_TEXT[cfg], "tokens_per_microbatch_per_gpu": T, "sim_ep": G,
                   "tokens_per_virtual_gpu": T // G, "top_k": K, "d_model": d, "ffn": F, "experts": E,
                   "placement": placement_desc,
                   "schedule": ("harmony" if layer.static_share is None
                                else f"harmony_pipelined (pipeline_ratio={args.pipeline_ratio})"),
                   "zipf_s": args.skew, "pass": "forward",
                   "launch": "cuda-graph replay" if not args.eager and not args.profile else "eager",
                   "microbatches": f"{n_seen} warm-up (seen: placement decided on them) + {n_unseen} held-out "
                                   f"(timed, cycled), seeds 1000..{1000 + n_seen + n_unseen - 1}",
                   "l2": "inputs larger than L2 (x %.0f MB per micro-batch, expert weights %.2f GB per step)"
                         % (T * d * 2 / 1e6, 3 * E * d * F * 2 / 1e9)},
        "max_mean_gpu_load": statistics.mean(cur),
        "max_mean_gpu_load_max": max(cur),
        "max_mean_gpu_load_static_cayley": statistics.mean(sta),
        "balance_heldout": {"timed_placement": _stat(cur), "static_cayley": _stat(sta),
                            "protocol": "placement decided by the reference policy (adaptive.py:119-166) on the "
                                        "warm-up micro-batches' expert loads only; max/mean of the integerized "
                                        "per-GPU loads of each held-out micro-batch (device scheduler)"},
        "replacement": replacement,
        "m_exact_last": [m_num, m_den],
        "gpu_loads_last": gpu_load,
        "scheduler_us": sched_us,
        "stage_ms": stage_ms,
        "roofline": {
            "bound": "tensor", "kernel": "hep_moe_expert_ffn (tcgen05 SwiGLU grouped GEMM x2)",
            "achieved": ffn_tflops, "peak": tf_sus, "unit": "TFLOP/s", "frac": ffn_tflops / tf_sus,
            "frac_of_burst_peak": ffn_tflops / tf_burst, "ffn_sm_clock": ffn_clock,
            # dense bf16 tcgen05 rate at the clock the GEMMs ran at: 8192 flop/clk/SM x SMs
            "frac_of_peak_at_ffn_clock": (ffn_tflops / (8192 * L.hep_device_sm_count() * ffn_clock["mhz"] * 1e6 / 1e12)
                                          if ffn_clock else None),
            "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside back-to-back steps)",
            "algorithmic_flops_per_launch": ffn_flops,
            # minimal DRAM bytes of one launch: every weight once, X read, H written + read, Y written
            "algorithmic_bytes_per_launch": E * 3 * d * F * 2 + R * d * 2 * 2 + R * F * 2 * 2,
            "traffic": traffic.get("ffn", {}).get("bytes"), "traffic_source": traffic.get("source"),
            "per_expert_roofline": per_expert,
        },
        "hbm_kernels": hbm_block(hbm_b2b_before, (perm_ms, comb_ms, rg_ms), (perm_bytes, comb_bytes, rg_bytes), hbm,
                                 traffic, router_flops=2 * T * d * layer.e_pad, tf_burst=tf_burst),
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": T * d * 2,
                "d2h_bytes_per_step": T * d * 2},
        "gpu_launches_per_step": layer.launches_per_forward(T),
        "clocks": sampler.summary() if sampler else None,
        "warmup_microbatch_metrics": [
            {"index": m.index, "max_load": m.max_gpu_load, "balance_ratio": round(m.balance_ratio, 6),
             "a2a_intra": m.a2a_intra, "local": m.local_volume, "layer_us": round(m.layer_time, 1)}
            for m in warm_rows],
    }
    if primary and cfg == "mixtral" and layer.static_share is None and not args.profile and args.balance_sweep:
        res["balance_sweep"] = balance_sweep(layer, pl_static, shape, seen, unseen, (1.0, 1.5, 2.0), stream)
    if primary and not args.profile and not args.no_train:
        res["train_step"] = measure_train(layer.placement, bias, cfg, unseen, dev, steps)
    del layer, seen, unseen, bufs, static_ds
    gc.collect()
    torch.cuda.empty_cache()
    return res


def per_expert_roofline(rows_e, d, F, tf_sus, hbm, ffn_ms):
    """The FFN's floor when experts run one after another, each at its own bound: tensor
    (6*d*F flop per row at tf_sus TFLOP/s) or HBM (its three weight matrices once plus its
    rows' X in, H out and in, Y out at hbm GB/s), whichever is longer; ms and frac of ffn_ms."""
    t_tc = [6.0 * d * F * r / (tf_sus * 1e12) for r in rows_e]
    t_hbm = [(3.0 * d * F * 2 + r * (4.0 * d + 4.0 * F)) / (hbm * 1e9) for r in rows_e]
    live = [i for i, r in enumerate(rows_e) if r > 0]
    ms = 1e3 * sum(max(t_tc[i], t_hbm[i]) for i in live)
    return {"ms": ms, "frac": ms / ffn_ms, "hbm_bound_experts": sum(1 for i in live if t_tc[i] < t_hbm[i]),
            "experts_with_rows": len(live), "rows_min_max": [min(rows_e), max(rows_e)]}


def hbm_block(before, after, nbytes, hbm, traffic, router_flops=None, tf_burst=None):
    """hbm_kernels: algorithmic bytes / back-to-back launch time / HBM copy peak, measured
    before the timed region (the kernel's own rate) with the after-region figure beside.
    router_gate also carries its tensor-core side: the router GEMM's 2*T*d*E_pad flops (the
    DeepSeek-V3 shape sits at the ridge point: HBM time ~ tensor time)."""
    out = {}
    for i, (name, tkey) in enumerate((("permute", "permute"), ("combine", "combine"), ("router_gate", "router_gate"))):
        gbs = nbytes[i] / (before[i] / 1e3) / 1e9
        gbs_after = nbytes[i] / (after[i] / 1e3) / 1e9
        out[name] = {"GB/s": gbs, "frac": gbs / hbm, "us": 1e3 * before[i], "algorithmic_bytes": nbytes[i],
                     "after_timed_region": {"GB/s": gbs_after, "frac": gbs_after / hbm, "us": 1e3 * after[i]},
                     "traffic": traffic.get(tkey, {}).get("bytes")}
    if router_flops and tf_burst:
        us = out["router_gate"]["us"]
        t_hbm, t_tc = nbytes[2] / hbm / 1e3, router_flops / tf_burst / 1e6  # µs at each peak
        out["router_gate"]["tensor"] = {"flops": router_flops, "TFLOP/s": router_flops / us / 1e6,
                                        "frac_of_burst": router_flops / us / 1e6 / tf_burst}
        out["router_gate"]["roofline_us"] = {"hbm": t_hbm, "tensor": t_tc, "bound": "hbm" if t_hbm >= t_tc else "tensor",
                                             "frac_of_bound": max(t_hbm, t_tc) / us}
    out["timing"] = ("each kernel re-launched 20x back to back on a held-out micro-batch inside one CUDA graph, "
                     "median of 5 timed replays after 5 warm ones, median over 4 held-out micro-batches; permute / combine "
                     "before the timed region after a 2 s rest, the router before the warm-up steps (the kernels' rate at "
                     "the nominal clock) and right after it (after the power-capped FFN steps: the in-step rate)")
    out["peak_GB/s"] = hbm
    return out


def measure_train(placement, bias, cfg, xs, dev, steps):
    """Forward + backward of the training layer (same kernels, 64-row aligned expert
    blocks, pre-activations kept), reported beside the forward line."""
    import torch

    import paper_2511_16947_b200 as P

    E, K, d, F, T, G = CONFIGS[cfg]
    tl = P.MoELayer(placement, d, F, K, seed=0, gate_bias=bias, device=dev, train=True)
    dout = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(77), device=dev).to(torch.bfloat16)
    stream = torch.cuda.current_stream()
    for i in range(2):
        tl(xs[i % len(xs)])
        tl.backward_step(xs[i % len(xs)], dout)
    torch.cuda.synchronize()
    n_tr = max(3, steps // 5)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_tr)]
    fev = _events(n_tr, ("ffn",))
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0e.record(stream)
    for i in range(n_tr):
        x = xs[i % len(xs)]
        tl.run(x, tl.buffers(T), stream, events=fev[i])
        ev[i][0].record(stream)
        tl.backward_step(x, dout)
        ev[i][1].record(stream)
    t1e.record(stream)
    torch.cuda.synchronize()
    tl.check_status()
    tr_ms = t0e.elapsed_time(t1e) / n_tr
    info = {
        "tokens_per_s": T / (tr_ms / 1e3), "ms_per_step": tr_ms,
        "backward_ms": statistics.mean(a.elapsed_time(b) for a, b in ev),
        "expert_ffn_fwd_ms": statistics.mean(f["ffn"][0].elapsed_time(f["ffn"][1]) for f in fev),
        "launches_per_step": tl.launches_per_forward(T) + tl.launches_per_backward(T),
        "note": "forward + backward (dx, dWg, dW13, dW2) of the same layer, no optimizer; held-out micro-batches; "
                "backward = combine^T, SwiGLU dgrad x2 + wgrad x2 (tcgen05), router^T, permute^T",
        "steps": n_tr,
    }
    del tl
    gc.collect()
    torch.cuda.empty_cache()
    return info


OTHER_KEYS = ("value", "ms_per_step", "steps", "max_mean_gpu_load", "max_mean_gpu_load_max",
              "max_mean_gpu_load_static_cayley", "replacement", "scheduler_us", "stage_ms", "e2e",
              "gpu_launches_per_step")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--skew", type=float, default=1.0)
    ap.add_argument("--placement", default="adaptive", choices=["adaptive", "cayley"])
    ap.add_argument("--batches", type=int, default=16,
                    help="distinct micro-batches: the first half warm up / feed the adaptive policy, the second "
                         "half (held out) is timed")
    ap.add_argument("--other-configs", default="qwen3,dsv3",
                    help="also measure these configs (shorter) and fold them into the line ('' = none)")
    ap.add_argument("--other-steps", type=int, default=40)
    ap.add_argument("--no-balance-sweep", dest="balance_sweep", action="store_false")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true", help="skip the forward+backward training-step measurement")
    ap.add_argument("--no-stress-sweep", dest="stress_sweep", action="store_false",
                    help="skip BASELINE configs[4] (Zipf 0/1/2 x 4K/64K/1M tokens x G 2/4/8, Qwen3-shaped layer)")
    ap.add_argument("--pipeline-ratio", type=float, default=None,
                    help="harmony_pipelined: share of tokens through the exact scheduler (rest split statically)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 EP protocol with every rank on GPU 0 (host-staged collectives; a check, not a bench)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 token exchange: NVLink peer stores fused into the dispatch / GEMM kernels, or NCCL all-to-all-v")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a CUDA-graph replay")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/cpu legs)")
    ap.add_argument("--tune", default="",
                    help="library launch tuning for A/B runs, e.g. 'ffn_pair=0 raster_gm1=8' (hep_tuning_set)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2511_16947_b200 import _lib

    if args.tune:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from _tuning import apply as apply_tuning

        apply_tuning(args.tune)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.dist_backend == "gloo":  # protocol check, all ranks may share one GPU
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "gloo":  # collectives staged through the host
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    if world > 1:
        run_ep(args, world, rank, local, dev)
        return
    _lib.require_cuda()

    res = measure_config(args.config, args, dev, steps=args.steps, primary=True)
    others = {}
    if not args.profile:
        for c in [c.strip() for c in args.other_configs.split(",") if c.strip()]:
            if c == args.config or c not in CONFIGS:
                continue
            o = measure_config(c, args, dev, steps=args.other_steps, primary=False)
            others[c] = {k: o[k] for k in OTHER_KEYS}
            others[c]["roofline"] = {k: o["roofline"][k] for k in ("achieved", "peak", "unit", "frac",
                                                                   "frac_of_burst_peak", "traffic",
                                                                   "per_expert_roofline")}
            others[c]["hbm_kernels"] = {k: {"GB/s": v["GB/s"], "frac": v["frac"]}
                                        for k, v in o["hbm_kernels"].items() if isinstance(v, dict)}
            others[c]["workload"] = o["config"]["workload"]
    E, K, d, F, T, G = CONFIGS[args.config]
    cores, model = cpu_info()
    cpu_line = sched_base = None
    if not args.no_cpu_baseline and not args.profile:
        sample = args.cpu_sample or {"tiny": 1024, "mixtral": 128, "qwen3": 512, "dsv3": 128}[args.config]
        per, walls = [], []
        for i in range(3):
            t0 = time.perf_counter()
            pt, info = cpu_reference_step(args.config, args.skew, sample, seed=i)
            walls.append(time.perf_counter() - t0)
            per.append(pt)
        cpu_line = {"value": 1.0 / statistics.mean(per), "unit": "tokens/s", "cores": cores, "kind": "port",
                    "sample": f"{sample} tokens x 3 steps through the CPU restatement (router+top-K+SwiGLU FFN "
                              f"numpy fp32 on all host threads) + Dinic scheduler oracle on a full {G}x{E} "
                              f"micro-batch; tokens/s extrapolated from the sample; host: {model}",
                    "sample_step_wall_ms": [round(1e3 * w, 1) for w in walls], "extrapolated": True}
        sched_base = sched_cpu_baseline(["mixtral", "qwen3", "dsv3"])
    line = {
        "metric": METRIC, "value": res["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": res["config"],
    }
    for k, v in res.items():
        if k not in ("value", "ms_per_step", "steps", "config", "gpu_launches_per_step"):
            line[k] = v
    line["gpu_launches"] = res["gpu_launches_per_step"] * args.steps
    line["cpu_baseline"] = cpu_line
    line["scheduler_cpu_baseline"] = sched_base
    line["other_configs"] = others or None
    if args.stress_sweep and not args.profile:
        # BASELINE configs[4], after the timed region: router / scheduler / assignment / dispatch
        # per micro-batch (CUDA events over 20 back-to-back launches of each stage), exact max/mean
        # load, and the CPU reference scheduler (Dinic port, 1 core) on the same load matrix
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from stress_sweep import sweep_points

        t0 = time.perf_counter()
        pts = list(sweep_points([2, 4, 8], [0.0, 1.0, 2.0], [4096, 65536, 1048576], reps=20))
        line["stress_sweep"] = {
            "config": "BASELINE configs[4]: Qwen3-30B-A3B-shaped layer (E=128, K=8, d=2048), Zipf s x tokens per "
                      "micro-batch x G scheduling GPUs, simulated EP on one B200, Cayley placement",
            "columns": ["G", "zipf_s", "tokens", "router_gate_us", "sched_us", "assign_us", "dispatch_us",
                        "dispatch_GB/s", "max_mean_gpu_load", "cpu_reference_sched_us"],
            "rows": [[p[k] for k in ("G", "zipf_s", "tokens", "router_gate_us", "sched_us", "assign_us",
                                     "dispatch_us", "dispatch_GB/s", "max_mean_gpu_load", "cpu_reference_sched_us")]
                     for p in pts],
            "cpu_reference": "oracle/hep_oracle.c (the reference's Dinic scheduler + integerize + routing restated "
                             "in C), 1 core, same load matrix",
            "wall_s": round(time.perf_counter() - t0, 1),
        }
    line["tuning"] = _lib.get_tuning()
    print(json.dumps(line))


if __name__ == "__main__":
    main()
