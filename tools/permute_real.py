"""K5 permute on the real DeepSeek-V3-shaped row map (Zipf s=1 routing, scheduled
receive layout) vs a random row map of the same size, back to back, cool GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402
from paper_2511_16947_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "dsv3"
E, K, d, F, T, G = bench.CONFIGS[cfg]
pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=torch.tensor(P.zipf_gate_bias(E, 1.0, 0)))
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
b = layer.buffers(T)
layer(x)
torch.cuda.synchronize()
L = _lib.lib()
s = _lib.stream_handle()
maps = {"real": b.tok_row, "random": torch.randperm(T * K, device="cuda").to(torch.int32).view(T, K)}
for name, m in maps.items():
    for _ in range(3):
        L.hep_moe_permute(x.data_ptr(), m.data_ptr(), T, K, d, b.rows.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        L.hep_moe_permute(x.data_ptr(), m.data_ptr(), T, K, d, b.rows.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1000
    gbs = (T * d * 2 * (1 + K) + T * K * 4) / (us * 1e-6) / 1e9
    print(f"{cfg} {name:6s} {us:7.1f} us {gbs:6.0f} GB/s")
