"""A/B the fused router+gate kernel (hep_router_topk) at the bench shapes:
router tile heights (hep_tuning.router_tile_rows: 0 / 128 = 128-row tiles, 112 = the
all-SM split of 16384 tokens, ...) interleaved over rounds in one process, plus the unfused chain
(hep_gemm_bf16 + hep_gate_topk + hep_gate_chunk_counts) for reference.  Prints the
median µs per launch and algorithmic GB/s (x, Wg, logits, top-K) / HBM peak; checks
that every variant produces the same top-K, histogram and chunk counts.

    python tools/router_ab.py [--variants 0,128] [--rounds 5] [--hot]
    python tools/router_ab.py --variants "router_mc=1,router_mc=2,router_mc=4"
(a variant is a tile height or "field=value[;field=value]" of hep_tuning; "ws=1": through
hep_router_topk_ws, the histogram zeroed inside the kernel)
--hot: before each timed batch, run 20 ms of bf16 GEMMs (the FFN's power state)."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16947_b200 import _lib as L  # noqa: E402

SHAPES = {"mixtral": (16384, 4096, 8, 2), "qwen3": (32768, 2048, 128, 8), "dsv3": (16384, 7168, 256, 8)}
ap = argparse.ArgumentParser()
ap.add_argument("--variants", default="0,128")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--hot", action="store_true")
ap.add_argument("--diag", action="store_true", help="load libhep_diag.so (tools/build_diag.sh)")
ap.add_argument("--graph", action="store_true", help="time a CUDA graph of the iters launches (no host launch cost)")
ap.add_argument("--shapes", default="mixtral,qwen3,dsv3")
args = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6553.6}
if args.diag:
    L.LIB_PATH = os.path.join(ROOT, "paper_2511_16947_b200", "libhep_diag.so")
lib = L.lib()
s = L.stream_handle()
base = L.get_tuning()
ha = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16) if args.hot else None
for name in args.shapes.split(","):
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
    nbytes = T * d * 2 + e_pad * d * 2 + T * e_pad * 4 + T * K * 8

    sync = torch.zeros(4, dtype=torch.int32, device="cuda")
    use_ws = [False]

    def fused(s=s):
        if use_ws[0]:  # in-kernel histogram zeroing (self-resetting sync words)
            L.check(lib.hep_router_topk_ws(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G,
                                           lg.data_ptr(), idx.data_ptr(), w.data_ptr(), h.data_ptr(), c.data_ptr(),
                                           sync.data_ptr(), s), "router")
            return
        L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G, lg.data_ptr(),
                                    idx.data_ptr(), w.data_ptr(), h.data_ptr(), c.data_ptr(), s), "router")

    def unfused(s=s):
        lib.hep_gemm_bf16(x.data_ptr(), wg.data_ptr(), lg.data_ptr(), T, e_pad, d, 0, s)
        lib.hep_gate_topk(lg.data_ptr(), e_pad, b.data_ptr(), T, E, K, tps, G, idx.data_ptr(), w.data_ptr(),
                          h.data_ptr(), s)
        lib.hep_gate_chunk_counts(idx.data_ptr(), T, K, E, tps, G, c.data_ptr(), s)

    def parse_variant(v):
        if "=" not in v:
            return ("tile=" + v, {"router_tile_rows": int(v)})
        return (v, {kv.split("=")[0]: int(kv.split("=")[1]) for kv in v.split(";") if not kv.startswith("ws")})

    variants = [parse_variant(v) for v in args.variants.split(",")] + [("unfused", None)]
    res = {lab: [] for lab, _ in variants}
    outs = {}
    for r in range(args.rounds):
        for lab, tile in variants:
            if tile is not None:
                L.set_tuning(**{**base, **tile})
                use_ws[0] = "ws=1" in lab

            fn = fused if tile is not None else unfused
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            if lab not in outs:
                outs[lab] = (idx.clone(), h.clone(), c.clone(), lg.clone())
            if ha is not None:
                for _ in range(10):
                    ha @ ha
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if args.graph:
                gr = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                with torch.cuda.stream(cs):
                    sc = L.stream_handle()
                    gr.capture_begin()
                    for _ in range(args.iters):
                        fn(sc)
                    gr.capture_end()
                gr.replay()
                torch.cuda.synchronize()
                st.record()
                gr.replay()
                en.record()
                torch.cuda.synchronize()
            else:
                st.record()
                for _ in range(args.iters):
                    fn()
                en.record()
                torch.cuda.synchronize()
            res[lab].append(st.elapsed_time(en) / args.iters * 1000)
    L.set_tuning(**base)
    ref = outs["unfused"]
    for lab, _ in variants:
        us = statistics.median(res[lab])
        same = all(torch.equal(a, b_) for a, b_ in zip(outs[lab], ref))
        print(json.dumps({"shape": name, "variant": lab, "us": round(us, 2), "GB/s": round(nbytes / us / 1e3, 1),
                          "frac": round(nbytes / us / 1e3 / peaks["hbm_gbs"], 3), "same_as_unfused": same,
                          "hot": args.hot, "all_us": [round(v, 1) for v in res[lab]]}))
