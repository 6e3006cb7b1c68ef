"""Time the K5 permute (one warp per token, 128-bit LSU copies) at the bench shapes on a
random row map, and check the rows it writes.  (A TMA bulk-copy variant — cp.async.bulk
row loads into shared memory, K bulk stores per row, 6 rows in flight per CTA — measured
5.52-5.75 TB/s against 5.76-5.82 TB/s here and was dropped, profiles/r01/ffn_ab_r01d.txt.)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16947_b200 import _lib as L  # noqa: E402

SHAPES = {"mixtral": (16384, 4096, 2), "qwen3": (32768, 2048, 8), "dsv3": (16384, 7168, 8)}
lib = L.lib()
s = L.stream_handle()
for name, (T, d, K) in SHAPES.items():
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    perm = torch.randperm(T * K, device="cuda").to(torch.int32).view(T, K)
    out = {}
    for impl in ("lsu",):
        rows = torch.zeros(T * K, d, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            lib.hep_moe_permute(x.data_ptr(), perm.data_ptr(), T, K, d, rows.data_ptr(), s)
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(20):
            lib.hep_moe_permute(x.data_ptr(), perm.data_ptr(), T, K, d, rows.data_ptr(), s)
        en.record()
        torch.cuda.synchronize()
        us = st.elapsed_time(en) / 20 * 1000
        gbs = (T * d * 2 * (1 + K) + T * K * 4) / (us * 1e-6) / 1e9
        out[impl] = rows
        print(f"{name:8s} {impl}: {us:7.1f} us  {gbs:6.0f} GB/s")
    assert torch.equal(out["lsu"][perm.view(-1).long()], x.repeat_interleave(K, dim=0)), name
print("rows ok")
