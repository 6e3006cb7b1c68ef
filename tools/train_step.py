"""One forward + backward of the training layer at a bench shape (for ncu launch lists):
    ncu --metrics gpu__time_duration.sum ... python tools/train_step.py --config mixtral"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--iters", type=int, default=2)
args = ap.parse_args()
E, K, d, F, T, G = bench.CONFIGS[args.config]
pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
bias = torch.tensor(P.zipf_gate_bias(E, 1.0, 0))
layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias, train=True)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
dout = torch.randn(T, d, device="cuda").to(torch.bfloat16)
for _ in range(args.iters):
    layer(x)
    layer.backward_step(x, dout)
torch.cuda.synchronize()
print("ok")
