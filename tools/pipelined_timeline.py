"""Event timeline of the pipelined split's dispatch chain (eager, two streams): every launch of
MoELayer.run's pipelined branch re-issued here with CUDA events around it on its stream.
    python tools/pipelined_timeline.py [config] [blocks_per_sm]
Prints (stream, stage, start µs, end µs) relative to the router's start, median of 5 runs."""
import ctypes
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_16947_b200 as P  # noqa: E402
from paper_2511_16947_b200 import _lib  # noqa: E402
from paper_2511_16947_b200.scheduler import HEP_SCHED_ALL  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen3"
bps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
E, K, d, F, T, G = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
layer = P.MoELayer(pl, d, F, K, seed=0, gate_bias=torch.tensor(P.zipf_gate_bias(E, 1.0, 0)), device=dev,
                   pipeline_ratio=0.5)
x = torch.randn(T, d, generator=torch.Generator(device=dev).manual_seed(1000), device=dev).to(torch.bfloat16)
layer(x)
torch.cuda.synchronize()
L = _lib.lib()
b = layer.buffers(T)
main = torch.cuda.Stream()
side = layer._side
tps = T // G
runs = []
for rep in range(6):
    evs = []

    def ev(stream, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append((stream is side, name, e))

    s, ss = main.cuda_stream, side.cuda_stream
    with torch.cuda.stream(main):
        ev(main, "router0")
        L.hep_router_topk_ws(x.data_ptr(), layer.wg.data_ptr(), T, d, E, layer.e_pad, _lib.ptr(layer.gate_bias), K, tps,
                             G, b.logits.data_ptr(), b.topk_idx.data_ptr(), b.topk_w.data_ptr(), b.hist.data_ptr(), None,
                             b.router_sync.data_ptr(), s)
        ev(main, "router1")
        layer.sched.launch_pipelined(b.hist, 1, E, layer.static_share, HEP_SCHED_ALL, main, stream_static=side)
        ev(main, "solve1")
        ev(side, "static_sched1")
        nnz = layer.sched.nnz
        split = layer.sched.split.data_ptr()
        L.hep_moe_assign_phase(layer.sched.handle, ctypes.byref(layer.sched.former.out), split, 0,
                               b.topk_idx.data_ptr(), T, K, tps, b.tok_row.data_ptr(), b.tok_row_ph[0].data_ptr(),
                               b.row_tok.data_ptr(), b.seg.data_ptr(), b.expert_rows.data_ptr(), b.assign_ws2.data_ptr(),
                               b.assign_ws2.numel(), ss)
        ev(side, "static_assign1")
        L.hep_moe_permute_ex(x.data_ptr(), b.tok_row_ph[0].data_ptr(), T, K, d, b.rows.data_ptr(), bps, ss)
        ev(side, "static_permute1")
        L.hep_moe_assign_phase(layer.sched.handle, ctypes.byref(layer.sched.out), split, 1, b.topk_idx.data_ptr(), T,
                               K, tps, b.tok_row.data_ptr(), b.tok_row_ph[1].data_ptr(), b.row_tok.data_ptr(),
                               b.seg.data_ptr() + 16 * nnz, b.expert_rows2.data_ptr(), b.assign_ws.data_ptr(),
                               b.assign_ws.numel(), s)
        ev(main, "sched_assign1")
        L.hep_moe_permute(x.data_ptr(), b.tok_row_ph[1].data_ptr(), T, K, d, b.rows.data_ptr(), s)
        ev(main, "sched_permute1")
        main.wait_stream(side)
        ev(main, "join")
    torch.cuda.synchronize()
    t0 = evs[0][2]
    runs.append({(sd, n): t0.elapsed_time(e) * 1e3 for sd, n, e in evs})
keys = list(runs[0])
print(cfg, "blocks/SM", bps)
for k in sorted(keys, key=lambda k: statistics.median(r[k] for r in runs[1:])):
    print(f"  {'side' if k[0] else 'main'} {k[1]:16s} {statistics.median(r[k] for r in runs[1:]):8.1f} us")
