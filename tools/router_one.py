"""Launch the fused router+gate (hep_router_topk) a few times at one bench shape, for
ncu captures:  python tools/router_one.py dsv3 [iters] [field=value ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16947_b200 import _lib as L  # noqa: E402

SHAPES = {"mixtral": (16384, 4096, 8, 2), "qwen3": (32768, 2048, 128, 8), "dsv3": (16384, 7168, 256, 8)}
name = sys.argv[1] if len(sys.argv) > 1 else "dsv3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
L.set_tuning(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[3:]})
T, d, E, K = SHAPES[name]
G = 8
e_pad = max(16, (E + 15) // 16 * 16)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
wg = (torch.randn(max(64, e_pad), d, device="cuda") / d ** 0.5).to(torch.bfloat16)
b = torch.randn(E, device="cuda")
tps = T // G
lg = torch.empty(T, e_pad, device="cuda")
idx = torch.empty(T, K, dtype=torch.int32, device="cuda")
w = torch.empty(T, K, device="cuda")
h = torch.empty(G, E, dtype=torch.int64, device="cuda")
c = torch.empty(G * (tps // 64) * E, dtype=torch.int32, device="cuda")
lib, s = L.lib(), L.stream_handle()
for _ in range(iters):
    L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G, lg.data_ptr(),
                                idx.data_ptr(), w.data_ptr(), h.data_ptr(), c.data_ptr(), s), "router")
torch.cuda.synchronize()
print(name, "ok", int(h.sum()))
