"""Per-CTA timeline of the fused router+gate kernel from a diagnostics build
(HEP_NVCC_DEFS=-DHEP_ROUTER_STAMPS, copied to libhep_diag.so):
    python tools/router_stamps.py [shape] [field=value ...]
Prints, over the CTAs of the last launch (µs from the first CTA's entry): entry spread,
last-MMA-issued, epilogue start / end, exit (median / max), and the launch's event time."""
import ctypes
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16947_b200 import _lib as L  # noqa: E402

L.LIB_PATH = os.path.join(ROOT, "paper_2511_16947_b200", "libhep_diag.so")
SHAPES = {"mixtral": (16384, 4096, 8, 2), "qwen3": (32768, 2048, 128, 8), "dsv3": (16384, 7168, 256, 8)}
names = [a for a in sys.argv[1:] if "=" not in a] or list(SHAPES)
# the stamps are compiled into the 1-CTA kernel only (router_pair=1; DSv3 would take the pair kernel)
L.set_tuning(**{"router_pair": 1, **{kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[1:] if "=" in kv}})
lib, s = L.lib(), L.stream_handle()
fn = lib.hep_diag_router_stamps
fn.argtypes = [ctypes.c_void_p]
for name in names:
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

    def run():
        L.check(lib.hep_router_topk(x.data_ptr(), wg.data_ptr(), T, d, E, e_pad, b.data_ptr(), K, tps, G, lg.data_ptr(),
                                    idx.data_ptr(), w.data_ptr(), h.data_ptr(), c.data_ptr(), s), "router")

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (256 * 8))()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record()
    run()
    q1.record()
    torch.cuda.synchronize()
    fn(ctypes.addressof(buf))
    st = [[buf[8 * i + j] for j in range(8)] for i in range(256)]
    n = min(T // 128, torch.cuda.get_device_properties(0).multi_processor_count)
    st = [r for r in st[:n] if r[0]]
    t0 = min(r[0] for r in st)
    col = lambda j: [(r[j] - t0) / 1e3 for r in st]  # noqa: E731
    out = {"shape": name, "ctas": len(st), "event_us": round(q0.elapsed_time(q1) * 1e3, 1)}
    for j, nm in enumerate(("entry", "last_mma", "epi_start", "epi_end", "exit", "pass1_end", "thresh_end", "pass2_end")):
        v = col(j)
        out[nm] = (round(statistics.median(v), 1), round(max(v), 1))
    print(out)
