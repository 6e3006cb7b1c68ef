"""BASELINE configs[4]: the scheduler + dispatch stress sweep — Zipf skew s in 0..2,
tokens 4K..1M per micro-batch, G = 2/4/8 scheduling GPUs (simulated EP on one B200).

For every point the MoE layer (Qwen3-30B-A3B shape: E=128, K=8, d=2048, F=768) runs
one forward, then each stage is re-launched back to back on that micro-batch (CUDA
events around 20 launches, so host launch latency does not enter): router + gate (K1)
µs, scheduler (K3) µs, token assignment (K4) µs, dispatch/permute (K5) µs and GB/s,
max/mean GPU load of the exact schedule, and the CPU reference scheduler (the Dinic
oracle port, C, one core) on the same load matrix for comparison.  One JSON object per
point on stdout.

    python tools/stress_sweep.py [--tokens 4096,65536,1048576] [--skews 0,0.5,1,1.5,2] [--gpus 2,4,8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sweep_points(gpus, skews, tokens, reps=20, cpu_reps=3):
    """Yield one dict per (G, s, T) point (see the module docstring)."""
    import ctypes

    import torch

    import paper_2511_16947_b200 as P
    from paper_2511_16947_b200 import _lib
    from oracle import oracle as O  # the CPU reference scheduler (checker / baseline only)

    L = _lib.lib()
    E, K, d, F = 128, 8, 2048, 768
    stages = ("router", "sched", "assign", "permute")
    for G in gpus:
        shape = P.ClusterShape(G, E, 2)
        pl = P.cayley_symmetric(shape)
        for s in skews:
            bias = torch.tensor(P.zipf_gate_bias(E, s, 0)) if s > 0 else None
            layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=bias)
            for T in tokens:
                T -= T % G
                x = torch.randn(T, d, generator=torch.Generator(device="cuda").manual_seed(T), device="cuda")
                x = x.to(torch.bfloat16)
                b = layer.buffers(T)
                layer.run(x, b)
                torch.cuda.synchronize()
                layer.check_status()
                st = torch.cuda.current_stream().cuda_stream
                tps = T // G
                launches = {
                    "router": lambda: L.hep_router_topk(x.data_ptr(), layer.wg.data_ptr(), T, d, E, layer.e_pad,
                                                        _lib.ptr(layer.gate_bias), K, tps, G, b.logits.data_ptr(),
                                                        b.topk_idx.data_ptr(), b.topk_w.data_ptr(), b.hist.data_ptr(),
                                                        b.assign_ws.data_ptr() + b.chunk_off, st),
                    "sched": lambda: layer.sched.launch_solve(b.hist, 1, E, None, 15),
                    "assign": lambda: L.hep_moe_assign_precounted(
                        layer.sched.handle, ctypes.byref(layer.sched.out), b.topk_idx.data_ptr(), T, K, tps,
                        b.row_align, b.tok_row.data_ptr(), b.row_tok.data_ptr(), b.seg.data_ptr(),
                        b.expert_rows.data_ptr(), b.assign_ws.data_ptr(), b.assign_ws.numel(), st),
                    "permute": lambda: L.hep_moe_permute(x.data_ptr(), b.tok_row.data_ptr(), T, K, d,
                                                         b.rows.data_ptr(), st),
                }
                ms = {}
                for k in stages:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    launches[k]()
                    e0.record()
                    for _ in range(reps):
                        launches[k]()
                    e1.record()
                    torch.cuda.synchronize()
                    ms[k] = e0.elapsed_time(e1) / reps
                layer.check_status()
                gl = layer.sched.gpu_load.cpu().tolist()
                mean = sum(gl) / len(gl)
                loads = b.hist.cpu().numpy().T.copy()  # [E][G] load matrix of this micro-batch
                t0 = time.perf_counter()
                for _ in range(cpu_reps):
                    O.full_path(G, pl.edp_groups, loads)
                cpu_us = (time.perf_counter() - t0) / cpu_reps * 1e6
                perm_bytes = T * d * 2 * (1 + K) + T * K * 4
                yield {
                    "G": G, "zipf_s": s, "tokens": T, "E": E, "K": K, "d_model": d,
                    "sched_us": round(1e3 * ms["sched"], 1), "assign_us": round(1e3 * ms["assign"], 1),
                    "router_gate_us": round(1e3 * ms["router"], 1),
                    "dispatch_us": round(1e3 * ms["permute"], 1),
                    "dispatch_GB/s": round(perm_bytes / (ms["permute"] / 1e3) / 1e9, 1),
                    "max_mean_gpu_load": round(max(gl) / mean, 4) if mean else 1.0,
                    "cpu_reference_sched_us": round(cpu_us, 1),
                }
                del x, b
                layer._bufs.clear()
            del layer
            torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="4096,16384,65536,262144,1048576")
    ap.add_argument("--skews", default="0,0.5,1,1.5,2")
    ap.add_argument("--gpus", default="2,4,8")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    for rec in sweep_points([int(v) for v in args.gpus.split(",")], [float(v) for v in args.skews.split(",")],
                            [int(v) for v in args.tokens.split(",")], args.reps):
        rec["cpu_reference"] = "Dinic oracle port (C, 1 core) on the same load matrix"
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
