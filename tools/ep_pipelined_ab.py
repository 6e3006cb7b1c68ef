"""A/B of the EP layer with and without the pipelined split, all G ranks in this process
(LocalComm: the all-to-all-v are device copies, the ranks' kernels share one GPU):
    python tools/ep_pipelined_ab.py [--configs qwen3,dsv3] [--ratio 0.5] [--rounds 5]
Also the plain layer without the per-slot regrouping of the received rows.
Prints ms per EP forward (host wall clock around forward + synchronize, median of rounds;
the NCCL path reads split sizes on the host, so the forward cannot be graph-captured) and
checks the outputs are identical."""
import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402
from paper_2511_16947_b200.ep import EPMoELayer, LocalComm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="qwen3,dsv3")
ap.add_argument("--ratio", type=float, default=0.5)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--p2p", action="store_true", help="the NVLink peer-store exchange with and without regrouping instead")
args = ap.parse_args()
dev = torch.device("cuda", 0)
for cfg in args.configs.split(","):
    E, K, d, F, T, G = bench.CONFIGS[cfg]
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
    x = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(1000), device=dev).to(torch.bfloat16)
    xs = [x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)]
    layers = {"plain": EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=0, gate_bias=bias)}
    if not args.p2p:  # (DeepSeek-V3: each 8-rank layer holds 45 GB of expert weights)
        layers["plain, no regroup"] = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=0, gate_bias=bias)
        layers["plain, no regroup"].regroup_rows = False
        layers[f"pipelined {args.ratio}"] = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=0, gate_bias=bias,
                                                       pipeline_ratio=args.ratio)
    else:
        layers["p2p"] = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=0, gate_bias=bias, exchange="p2p")
        layers["p2p, no regroup"] = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=0, gate_bias=bias,
                                               exchange="p2p")
        layers["p2p, no regroup"].regroup_rows = False
    outs, res = {}, {k: [] for k in layers}
    for k, lay in layers.items():
        for _ in range(2):
            o = lay.forward(xs)
        torch.cuda.synchronize()
        outs[k] = torch.cat([t.clone() for t in o])
    for _ in range(args.rounds):
        for k, lay in layers.items():
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.iters):
                lay.forward(xs)
            torch.cuda.synchronize()
            res[k].append((time.perf_counter() - t0) * 1e3 / args.iters)
    ref = outs["plain"]
    for k in layers:
        print(json.dumps({"config": cfg, "variant": k, "G": G, "ms": round(statistics.median(res[k]), 3),
                          "all_ms": [round(v, 3) for v in res[k]], "same_as_plain": bool(torch.equal(outs[k], ref))}))
    del layers
    torch.cuda.empty_cache()
