"""Time the fused router+gate kernel (hep_router_topk) against the unfused chain
(hep_gemm_bf16 + hep_gate_topk + hep_gate_chunk_counts) at the bench shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16947_b200 import _lib as L  # noqa: E402

SHAPES = {"mixtral": (16384, 4096, 8, 2), "qwen3": (32768, 2048, 128, 8), "dsv3": (16384, 7168, 256, 8)}
lib = L.lib()
s = L.stream_handle()
for name, (T, d, E, K) in SHAPES.items():
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

    def fused(logits=True):
        lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G,
                            lg.data_ptr() if logits else None, idx.data_ptr(), w.data_ptr(), h.data_ptr(),
                            c.data_ptr(), s)

    def unfused():
        lib.hep_gemm_bf16(x.data_ptr(), wg.data_ptr(), lg.data_ptr(), T, e_pad, d, 0, s)
        lib.hep_gate_topk(lg.data_ptr(), e_pad, b.data_ptr(), T, E, K, tps, G, idx.data_ptr(), w.data_ptr(),
                          h.data_ptr(), s)
        lib.hep_gate_chunk_counts(idx.data_ptr(), T, K, E, tps, G, c.data_ptr(), s)

    def gemm_only():
        lib.hep_gemm_bf16(x.data_ptr(), wg.data_ptr(), lg.data_ptr(), T, e_pad, d, 0, s)

    for label, fn in (("fused", fused), ("fused_nologits", lambda: fused(False)), ("unfused", unfused),
                      ("gemm_only", gemm_only)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(50):
            fn()
        en.record()
        torch.cuda.synchronize()
        print(f"{name:8s} {label:15s} {st.elapsed_time(en) / 50 * 1000:8.1f} us")
