"""A/B env knobs on the training layer's backward (`MoELayer.backward_step`) in one
process, interleaved rounds, CUDA-event time per backward; checks the gradients of
every variant match the first's (bit-pattern fingerprints).

    python tools/bwd_ab.py --config qwen3 --variants "HEP_ST256=0;HEP_ST256=1"
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3")
ap.add_argument("--variants", default="HEP_ST256=0;HEP_ST256=1")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--rounds", type=int, default=6)
args = ap.parse_args()
E, K, d, F, T, G = bench.CONFIGS[args.config]
pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=torch.tensor(P.zipf_gate_bias(E, 1.0, 0)), train=True)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
dout = torch.randn(T, d, device="cuda").to(torch.bfloat16)
layer(x)
variants = [v.strip() for v in args.variants.split(";")]
from _tuning import apply as apply_tuning  # noqa: E402
from paper_2511_16947_b200 import _lib  # noqa: E402

base = _lib.get_tuning()
res = {v: [] for v in variants}
grads = {}
for r in range(args.rounds):
    for v in variants:
        apply_tuning(v, base)
        g = layer.backward_step(x, dout)
        torch.cuda.synchronize()
        if v not in grads:
            # exact fingerprint per gradient (bit pattern sums; cloning DSv3's 42 GB would not fit)
            grads[v] = [int(t.contiguous().view(torch.int16 if t.element_size() == 2 else torch.int32).to(torch.int64).sum())
                        for t in (g if isinstance(g, (tuple, list)) else [g]) if torch.is_tensor(t)]
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(args.iters):
            layer.backward_step(x, dout)
        en.record()
        torch.cuda.synchronize()
        res[v].append(st.elapsed_time(en) / args.iters)
_lib.set_tuning(**base)
g0 = grads[variants[0]]
for v in variants:
    same = grads[v] == g0
    print(json.dumps({"config": args.config, "variant": v, "backward_ms": round(statistics.median(res[v]), 3),
                      "same_grads": same, "ms_all": [round(m, 3) for m in res[v]]}))
