"""In-process A/B of plain harmony vs the pipelined split (static share on a side stream) at
the bench shapes, interleaved over rounds, each layer captured as a CUDA graph:
    python tools/pipelined_ab.py [--configs qwen3,dsv3,mixtral] [--blocks 8,6,4] [--rounds 5]
Prints µs per layer step (median over rounds) and whether each variant's output is
bit-identical to the plain layer's."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="qwen3,dsv3,mixtral")
ap.add_argument("--blocks", default="8,6,4")
ap.add_argument("--ratio", type=float, default=0.5)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--dispatch-only", action="store_true", help="time the chain up to the permute only")
args = ap.parse_args()
dev = torch.device("cuda", 0)
for cfg in args.configs.split(","):
    E, K, d, F, T, G = bench.CONFIGS[cfg]
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    x = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(1000), device=dev).to(torch.bfloat16)
    plain = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias, device=dev)
    pipe = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias, device=dev, pipeline_ratio=args.ratio)
    variants = [("plain", plain, None)] + [(f"pipelined b/SM={b}", pipe, int(b)) for b in args.blocks.split(",")]
    graphs, outs = {}, {}
    for name, layer, bps in variants:
        if bps is not None:
            layer.static_permute_blocks_per_sm = bps
        graphs[name] = layer.capture(x, dispatch_only=args.dispatch_only)
        graphs[name].replay()
        torch.cuda.synchronize()
        outs[name] = layer.buffers(T).out.clone() if not args.dispatch_only else layer.buffers(T).rows.clone()
    res = {n: [] for n, _, _ in variants}
    for _ in range(args.rounds):
        for name, layer, bps in variants:
            g = graphs[name]
            g.replay()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            for _ in range(args.iters):
                g.replay()
            q1.record()
            torch.cuda.synchronize()
            res[name].append(q0.elapsed_time(q1) / args.iters * 1e3)
    ref = outs["plain"]
    for name, _, bps in variants:
        print(json.dumps({"config": cfg, "variant": name, "us": round(statistics.median(res[name]), 1),
                          "all_us": [round(v, 1) for v in res[name]],
                          "same_as_plain": bool(torch.equal(outs[name], ref)) if not args.dispatch_only else None}))
    del plain, pipe, graphs
    torch.cuda.empty_cache()
