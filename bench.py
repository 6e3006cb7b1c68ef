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
    for _ in range(args.warmup):
        cpu_reference_step(cfg, args.skew, max(8, sample // 8))
    per = []
    for i in range(args.steps):
        pt, info = cpu_reference_step(cfg, args.skew, sample, seed=i)
        per.append(pt)
    value = 1.0 / statistics.mean(per)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(per) * T,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": CONFIG_TEXT[cfg], "tokens_per_microbatch": T, "sim_ep": G, "top_k": K,
                   "zipf_s": args.skew},
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
    layer = EPMoELayer(pl, d, F, K, comm, [rank], seed=0, gate_bias=bias, device=dev, exchange=args.exchange)
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
                       "launch": ("cuda-graph replay (device-side barriers, no host sync)" if graph is not None
                                  else "eager"),
                       "exchange": (("NVLink peer stores: dispatch kernel -> peers' receive buffers, down-projection "
                                     "epilogue -> sources' return buffers (CUDA IPC); histogram all-gather + 2 barriers")
                                    if args.exchange == "p2p" else
                                    ("NCCL" if args.dist_backend == "nccl" else "gloo, host-staged (protocol check)")
                                    + " all-gather (histograms) + all-to-all-v dispatch/combine")},
            "max_mean_gpu_load": mm, "max_mean_gpu_load_static_cayley": static_mm, "replacement": replacement,
            "e2e": {"value": world * T * args.steps / (e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": T * d * 2, "d2h_bytes_per_step": T * d * 2},
            "gpu_launches": args.steps * (13 if args.exchange == "p2p" else 12),
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
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--skew", type=float, default=1.0)
    ap.add_argument("--placement", default="adaptive", choices=["adaptive", "cayley"])
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true", help="skip the forward+backward training-step measurement")
    ap.add_argument("--pipeline-ratio", type=float, default=None,
                    help="harmony_pipelined: share of tokens through the exact scheduler (rest split statically)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 EP protocol with every rank on GPU 0 (host-staged collectives; a check, not a bench)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 token exchange: NVLink peer stores fused into the dispatch / GEMM kernels, or NCCL all-to-all-v")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a CUDA-graph replay")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/cpu legs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200 import _lib

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

    E, K, d, F, T, G = CONFIGS[args.config]
    if world > 1:
        run_ep(args, world, rank, local, dev)
        return
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, args.skew, 0)) if args.skew > 0 else None
    layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias, device=dev, pipeline_ratio=args.pipeline_ratio)
    gx = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(T, d, generator=gx, device=dev).to(torch.bfloat16)
    bufs = layer.buffers(T)
    stream = torch.cuda.current_stream()
    L = _lib.lib()

    def step():
        layer.run(x, layer.buffers(T), stream)

    def gpu_balance():
        gl = layer.sched.gpu_load.cpu().tolist()
        mean = sum(gl) / len(gl)
        return (max(gl) / mean if mean else 1.0), gl

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    layer.check_status()
    static_max_mean, static_loads = gpu_balance()
    placement_desc = f"cayley_symmetric(G={G}, E={E}, d=2)"
    replacement = None
    if args.placement == "adaptive":
        # the paper's adaptive replacement (adaptive.py:119-166): score the static
        # placement on the observed expert loads and adopt the greedy + Monte-Carlo
        # candidate when it is better; a one-off, off the per-micro-batch path
        from paper_2511_16947_b200.adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace

        hist = LoadHistory(8)
        hist.push(layer.expert_loads(T))
        dec = evaluate_and_maybe_replace(pl, hist, ReplacementPolicy(threshold=1.0, mc_samples=200), shape, 0)
        replacement = dec.to_event(args.warmup)
        if dec.replaced:
            layer.set_placement(dec.placement)
            placement_desc = (f"adaptive: greedy replica counts {list(P.placement.greedy_replica_counts(hist.entries[0], E * 2, max_count=G))}"
                              f" + Monte-Carlo layout (200 samples), from cayley_symmetric(G={G}, E={E}, d=2)")
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            layer.check_status()
    bufs = layer.buffers(T)

    # --- timed region: K steps back to back; per-stage events on the launching stream
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    stages = ("router", "gate", "sched", "assign", "permute", "ffn", "combine")
    evs = [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in stages}
           for _ in range(args.steps)]

    def staged_step(i):
        layer.run(x, bufs, stream, events=evs[i])

    # the timed step is one CUDA-graph replay of the whole forward (11 kernels, no host
    # sync); per-stage times come from an eager pass with events around each stage
    graph = None
    if not args.profile and not args.eager:
        try:
            graph = layer.capture(x)
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # capture is an optimisation; eager launches are the same kernels
            print(f"[bench] CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graph = None
    sampler = ClockSampler(local) if not args.profile else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    start.record(stream)
    for i in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            staged_step(i)
    end.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    if world > 1:
        dist.barrier()
    layer.check_status()
    t_ms = start.elapsed_time(end)
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = world * T * args.steps / (t_ms / 1e3)
    if graph is not None:  # stage breakdown from eager steps
        for i in range(args.steps):
            staged_step(i)
        torch.cuda.synchronize()

    stage_ms = {k: statistics.mean(e[k][0].elapsed_time(e[k][1]) for e in evs) for k in stages}
    ffn_ms, perm_ms, comb_ms = stage_ms["ffn"], stage_ms["permute"], stage_ms["combine"]

    # --- the SM clock the expert GEMMs actually ran at: CTA 0 stamps clock64 and the
    # global timer at entry/exit of each GEMM (hep_tuning.ffn_clock = 1), eager steps back to back
    ffn_clock = None
    if not args.profile:
        import ctypes as _ct

        with _lib.tuning(ffn_clock=1):
            for i in range(min(args.steps, 10)):
                staged_step(i)
            torch.cuda.synchronize()
            st = (_ct.c_int64 * 8)()
            _lib.check(L.hep_ffn_debug_clock(st), "hep_ffn_debug_clock")
            mhz = [1e3 * (st[4 * g + 2] - st[4 * g]) / max(1, st[4 * g + 3] - st[4 * g + 1]) for g in range(2)]
            ns = [st[4 * g + 3] - st[4 * g + 1] for g in range(2)]
            ffn_clock = {"gemm1_mhz": round(mhz[0], 1), "gemm2_mhz": round(mhz[1], 1),
                         "mhz": round((mhz[0] * ns[0] + mhz[1] * ns[1]) / max(1, ns[0] + ns[1]), 1),
                         "source": "clock64 / globaltimer of CTA 0 across each expert GEMM (eager steps)"}

    # --- scheduler latency: the K3 kernel alone, on this micro-batch's histogram
    n_sched = 200
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(n_sched):
        layer.sched.launch_solve(bufs.hist, 1, E, None, 15, stream)
    s1.record(stream)
    torch.cuda.synchronize()
    sched_us = 1e3 * s0.elapsed_time(s1) / n_sched

    # --- the HBM-bound kernels re-launched back to back on this micro-batch (they are
    # idempotent), so the host's eager launch latency does not enter their bandwidth
    def _b2b_ms(fn, n=20):
        fn()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(n):
            fn()
        q1.record(stream)
        torch.cuda.synchronize()
        return q0.elapsed_time(q1) / n

    tps = T // G
    perm_ms = _b2b_ms(lambda: _lib.check(L.hep_moe_permute(x.data_ptr(), bufs.tok_row.data_ptr(), T, K, d,
                                                           bufs.rows.data_ptr(), stream.cuda_stream), "permute"))
    comb_ms = _b2b_ms(lambda: _lib.check(L.hep_moe_combine(bufs.y.data_ptr(), bufs.tok_row.data_ptr(),
                                                           bufs.topk_w.data_ptr(), T, K, d, bufs.out.data_ptr(),
                                                           stream.cuda_stream), "combine"))
    chunk = None if layer.static_share is not None else bufs.assign_ws.data_ptr() + bufs.chunk_off
    rg_ms = _b2b_ms(lambda: _lib.check(L.hep_router_topk(
        x.data_ptr(), layer.wg.data_ptr(), T, d, E, layer.e_pad, _lib.ptr(layer.gate_bias), K, tps, G,
        bufs.logits.data_ptr(), bufs.topk_idx.data_ptr(), bufs.topk_w.data_ptr(), bufs.hist.data_ptr(), chunk,
        stream.cuda_stream), "router"))
    torch.cuda.synchronize()
    layer.check_status()

    gpu_load = layer.sched.gpu_load.cpu().tolist()
    m_num, m_den = layer.sched.m[:2].cpu().tolist()
    mean_load = sum(gpu_load) / len(gpu_load)
    max_mean = max(gpu_load) / mean_load if mean_load else 1.0

    # --- e2e through the public API with host buffers (pinned): every step copies
    # its input batch host->device and its output device->host inside the timed
    # region (HostPipeline overlaps batch i+1's H2D and batch i-1's D2H with batch i)
    from paper_2511_16947_b200.layer import HostPipeline

    pipe = HostPipeline(layer, T)
    xh = [x.cpu().pin_memory() for _ in range(2)]
    for i in range(3):
        pipe.submit(xh[i % 2])
    pipe.drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_in)
    last = None
    for i in range(args.steps):
        last = pipe.submit(xh[i % 2])
    out_last = pipe.result(last)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(pipe.s_out)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    e_wall = (time.perf_counter() - t0) * 1e3
    e_ms = max(e_ms, e_wall)  # device span from first H2D to last D2H, never below the host clock
    if world > 1:
        tt = torch.tensor([e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_ms = float(tt.item())
    e2e_value = world * T * args.steps / (e_ms / 1e3)
    assert torch.isfinite(out_last.float()).all()

    # --- training step (forward + backward through the same kernels), reported beside
    train_info = None
    if not args.profile and not args.no_train:
        del pipe
        tl = P.MoELayer(layer.placement, d, F, K, seed=0, gate_bias=bias, device=dev, train=True)
        dout = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(77), device=dev).to(torch.bfloat16)
        for _ in range(2):
            tl(x)
            tl.backward_step(x, dout)
        torch.cuda.synchronize()
        n_tr = max(3, args.steps // 5)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_tr)]
        fev = [{"ffn": (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))} for _ in range(n_tr)]
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(stream)
        for i in range(n_tr):
            tl.run(x, tl.buffers(T), stream, events=fev[i])
            ev[i][0].record(stream)
            tl.backward_step(x, dout)
            ev[i][1].record(stream)
        t1e.record(stream)
        torch.cuda.synchronize()
        tl.check_status()
        tr_ms = t0e.elapsed_time(t1e) / n_tr
        bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
        ffn_f = statistics.mean(f["ffn"][0].elapsed_time(f["ffn"][1]) for f in fev)
        train_info = {
            "tokens_per_s": T / (tr_ms / 1e3),
            "ms_per_step": tr_ms,
            "backward_ms": bwd_ms,
            "expert_ffn_fwd_ms": ffn_f,
            "note": "forward + backward (dx, dWg, dW13, dW2) of the same layer, no optimizer; "
                    "backward = combine^T, SwiGLU dgrad x2 + wgrad x2 (tcgen05), router^T, permute^T",
            "steps": n_tr,
        }
        del tl
        torch.cuda.empty_cache()

    hbm, tf_burst, tf_sus, peak_src = load_peaks()
    traffic = load_traffic(args.config)
    R = T * K
    ffn_flops = 6.0 * d * F * R
    ffn_tflops = ffn_flops / (ffn_ms / 1e3) / 1e12
    perm_bytes = T * d * 2 * (1 + K) + T * K * 4
    comb_bytes = T * K * d * 2 + T * K * 4 * 2 + T * d * 2
    rg_bytes = T * d * 2 + layer.e_pad * d * 2 + T * layer.e_pad * 4 + T * K * 8  # x, Wg, logits, top-K
    launches_per_step = layer.launches_per_forward(T)

    if rank == 0:
        cores, model = cpu_info()
        cpu_line = None
        if not args.no_cpu_baseline and not args.profile:
            sample = args.cpu_sample or {"tiny": 1024, "mixtral": 128, "qwen3": 512, "dsv3": 128}[args.config]
            per = []
            for i in range(3):
                pt, info = cpu_reference_step(args.config, args.skew, sample, seed=i)
                per.append(pt)
            cpu_line = {"value": 1.0 / statistics.mean(per), "unit": "tokens/s", "cores": cores, "kind": "port",
                        "sample": f"{sample} tokens x 3 steps through the CPU restatement (router+top-K+SwiGLU FFN "
                                  f"numpy fp32 on all host threads) + Dinic scheduler oracle on a full {G}x{E} "
                                  f"micro-batch; host: {model}"}
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": CONFIG_TEXT[args.config],
                "tokens_per_microbatch_per_gpu": T,
                "sim_ep": G,
                "tokens_per_virtual_gpu": T // G,
                "top_k": K, "d_model": d, "ffn": F, "experts": E,
                "placement": placement_desc,
                "schedule": ("harmony" if args.pipeline_ratio is None
                             else f"harmony_pipelined (pipeline_ratio={args.pipeline_ratio})"),
                "zipf_s": args.skew,
                "pass": "forward",
                "launch": "cuda-graph replay" if graph is not None else "eager",
                "l2": "inputs larger than L2 (x %.0f MB, expert weights %.2f GB per step)" % (T * d * 2 / 1e6,
                                                                                               3 * E * d * F * 2 / 1e9),
            },
            "max_mean_gpu_load": max_mean,
            "max_mean_gpu_load_static_cayley": static_max_mean,
            "replacement": replacement,
            "m_exact": [m_num, m_den],
            "gpu_loads": gpu_load,
            "scheduler_us": sched_us,
            "stage_ms": stage_ms,
            "roofline": {
                "bound": "tensor",
                "kernel": "hep_moe_expert_ffn (tcgen05 SwiGLU grouped GEMM x2)",
                "achieved": ffn_tflops,
                "peak": tf_sus,
                "unit": "TFLOP/s",
                "frac": ffn_tflops / tf_sus,
                "frac_of_burst_peak": ffn_tflops / tf_burst,
                # dense bf16 tcgen05 rate at the clock the GEMMs ran at: 8192 flop/clk/SM x 148 SMs
                "ffn_sm_clock": ffn_clock,
                "frac_of_peak_at_ffn_clock": (ffn_tflops / (8192 * L.hep_device_sm_count() * ffn_clock["mhz"] * 1e6 / 1e12)
                                              if ffn_clock else None),
                "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside back-to-back steps)",
                "algorithmic_flops_per_launch": ffn_flops,
                # minimal DRAM bytes of one launch: every weight once, X read, H written + read, Y written
                "algorithmic_bytes_per_launch": E * 3 * d * F * 2 + R * d * 2 * 2 + R * F * 2 * 2,
                "traffic": traffic.get("ffn", {}).get("bytes"),
                "traffic_source": traffic.get("source"),
            },
            "hbm_kernels": {
                "permute": {"GB/s": perm_bytes / (perm_ms / 1e3) / 1e9, "frac": perm_bytes / (perm_ms / 1e3) / 1e9 / hbm,
                            "algorithmic_bytes": perm_bytes, "traffic": traffic.get("permute", {}).get("bytes")},
                "combine": {"GB/s": comb_bytes / (comb_ms / 1e3) / 1e9, "frac": comb_bytes / (comb_ms / 1e3) / 1e9 / hbm,
                            "algorithmic_bytes": comb_bytes, "traffic": traffic.get("combine", {}).get("bytes")},
                # K1 fused router GEMM + gate: reads x and Wg, writes logits, top-K, weights
                "router_gate": {"GB/s": rg_bytes / (rg_ms / 1e3) / 1e9, "frac": rg_bytes / (rg_ms / 1e3) / 1e9 / hbm,
                                "algorithmic_bytes": rg_bytes, "traffic": traffic.get("router_gate", {}).get("bytes")},
                "timing": "each kernel re-launched 20x back to back on the step's data, CUDA events",
                "peak_GB/s": hbm,
            },
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": T * d * 2,
                    "d2h_bytes_per_step": T * d * 2},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": sampler.summary() if sampler else None,
            "cpu_baseline": cpu_line,
            "train_step": train_info,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
