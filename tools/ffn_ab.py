"""A/B the expert-FFN kernel variants in ONE process, interleaved, with time AND
energy per launch (the FFN-heavy configs run power-capped, so joules per step
decide the achieved clock).

    python tools/ffn_ab.py --config dsv3 --variants "HEP_FFN_PAIR=0;HEP_FFN_PAIR=1" [--iters 30 --rounds 4]

The layer is built and placed as in bench.py (Zipf s=1 gate bias; adaptive
replacement when it beats Cayley), one forward fills the receive rows, then
each variant launches `hep_moe_expert_ffn` `iters` times back to back; the
variants cycle `rounds` times.  Variants are applied with hep_tuning_set (tools/_tuning.py),
read by the library at every call, so they switch in-process.  Prints one JSON line per variant.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv3")
    ap.add_argument("--variants", default="HEP_FFN_PAIR=1")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--skew", type=float, default=1.0)
    ap.add_argument("--placement", default="adaptive", choices=["adaptive", "cayley"])
    ap.add_argument("--diag", action="store_true", help="load libhep_diag.so (a diagnostics build)")
    args = ap.parse_args()

    import torch
    import pynvml

    import bench
    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200 import _lib

    if args.diag:
        _lib.LIB_PATH = os.path.join(ROOT, "paper_2511_16947_b200", "libhep_diag.so")

    E, K, d, F, T, G = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    shape = P.ClusterShape(G, E, 2)
    pl = P.cayley_symmetric(shape)
    bias = torch.tensor(P.zipf_gate_bias(E, args.skew, 0)) if args.skew > 0 else None
    layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias, device=dev)
    x = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(1000), device=dev).to(torch.bfloat16)
    layer(x)
    torch.cuda.synchronize()
    if args.placement == "adaptive":
        from paper_2511_16947_b200.adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace

        hist = LoadHistory(8)
        hist.push(layer.expert_loads(T))
        dec = evaluate_and_maybe_replace(pl, hist, ReplacementPolicy(threshold=1.0, mc_samples=200), shape, 0)
        if dec.replaced:
            layer.set_placement(dec.placement)
    layer(x)
    torch.cuda.synchronize()
    b = layer.buffers(T)
    L = _lib.lib()
    s = torch.cuda.current_stream()
    flops = 6.0 * d * F * b.R

    def ffn():
        if os.environ.get("AB_GATHER") == "1":  # permute fused into GEMM 1 (TMA gather of x rows)
            _lib.check(L.hep_moe_expert_ffn_gather(x.data_ptr(), T, b.row_tok.data_ptr(), layer.w13.data_ptr(),
                                                   layer.w2.data_ptr(), b.seg.data_ptr(), b.n_seg, b.R, d, F, E,
                                                   b.h.data_ptr(), b.y.data_ptr(), b.ffn_ws.data_ptr(),
                                                   b.ffn_ws.numel(), layer.sched.status.data_ptr(), s.cuda_stream),
                       "ffn_gather")
            return
        _lib.check(L.hep_moe_expert_ffn(b.rows.data_ptr(), layer.w13.data_ptr(), layer.w2.data_ptr(), b.seg.data_ptr(),
                                        b.n_seg, b.R, d, F, E, b.h.data_ptr(), b.y.data_ptr(), b.ffn_ws.data_ptr(),
                                        b.ffn_ws.numel(), layer.sched.status.data_ptr(), s.cuda_stream), "ffn")

    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    variants = [v.strip() for v in args.variants.split(";")]
    res = {v: {"ms": [], "J": [], "mhz": []} for v in variants}
    from _tuning import apply as apply_tuning

    base_tuning = _lib.get_tuning()
    ref_y = {}
    for _ in range(3):
        ffn()
    torch.cuda.synchronize()
    for r in range(args.rounds):
        for v in variants:
            apply_tuning(v, base_tuning)
            for _ in range(3):
                ffn()
            torch.cuda.synchronize()
            if v not in ref_y:
                ref_y[v] = b.y.clone()
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hnd)
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.record(s)
            for i in range(args.iters):
                ffn()
                if i == args.iters // 2:
                    mhz = pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
            en.record(s)
            torch.cuda.synchronize()
            e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hnd)
            ms = st.elapsed_time(en) / args.iters
            res[v]["ms"].append(ms)
            res[v]["J"].append((e1 - e0) / 1000.0 / args.iters)
            res[v]["mhz"].append(mhz)
    _lib.set_tuning(**base_tuning)
    y0 = ref_y[variants[0]]
    for v in variants:
        ms = statistics.median(res[v]["ms"])
        print(json.dumps({"config": args.config, "variant": v, "ffn_ms": round(ms, 4),
                          "TF/s": round(flops / ms / 1e9, 1), "J_per_ffn": round(statistics.median(res[v]["J"]), 3),
                          "sm_mhz": statistics.median(res[v]["mhz"]), "rows": b.R,
                          "same_as_first": bool(torch.equal(ref_y[v], y0)), "ms_all": [round(m, 3) for m in res[v]["ms"]]}))


if __name__ == "__main__":
    main()
