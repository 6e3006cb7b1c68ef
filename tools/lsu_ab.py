"""A/B the 128-bit vs 256-bit LSU permute (K5) kernel (hep_tuning.lsu256 = 0/1, read per
call) at the bench shapes on a random row map, interleaved rounds; checks both
variants write identical bytes.  (A 256-bit combine measured 5-10 % slower and was
dropped, profiles/r01/ab_lsu_r01i.txt; the combine rows here time the kept kernel.)"""
import json
import os
import statistics
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
    w = torch.rand(T, K, device="cuda")
    rows = torch.empty(T * K, d, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    ops = {
        "permute": (lambda: lib.hep_moe_permute(x.data_ptr(), perm.data_ptr(), T, K, d, rows.data_ptr(), s),
                    T * d * 2 * (1 + K) + T * K * 4),
        "combine": (lambda: lib.hep_moe_combine(rows.data_ptr(), perm.data_ptr(), w.data_ptr(), T, K, d,
                                                out.data_ptr(), s), T * d * 2 * (1 + K) + T * K * 8),
    }
    for op, (fn, nbytes) in ops.items():
        res, ref = {"0": [], "1": []}, {}
        for r in range(10):
            for v in ("0", "1"):
                L.set_tuning(lsu256=int(v))
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                ref.setdefault(v, (rows if op == "permute" else out).clone())
                st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                st.record()
                for _ in range(20):
                    fn()
                en.record()
                torch.cuda.synchronize()
                res[v].append(st.elapsed_time(en) / 20 * 1000)
        for v in ("0", "1"):
            us = statistics.median(res[v])
            print(json.dumps({"shape": name, "op": op, "lsu256": v, "us": round(us, 1),
                              "GB/s": round(nbytes / us / 1e3, 0), "same": bool(torch.equal(ref[v], ref["0"]))}))
