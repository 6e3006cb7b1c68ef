"""Small-shape run of every hot-path kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py

Covers: fused router+gate (one and two epilogue column halves, 64-aligned and
chunk-straddling tiles, CTA pairs, in-kernel histogram zeroing), the scheduler (solve / integerize / route / transfer,
pipelined split on two streams), the assignment kernels, permute (128/256-bit),
the expert FFN (1-CTA and CTA-pair grouped GEMMs, light-expert split), combine,
the backward (dgrad / K-ragged wgrad / router backward), and the EP exchange
over peer stores with all ranks in one process (dispatch, return addresses,
the down-projection epilogue storing into the sources' buffers, rows regrouped per slot)
and the EP pipelined split."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_16947_b200 as P  # noqa: E402
from paper_2511_16947_b200 import _lib  # noqa: E402
from paper_2511_16947_b200.ep import EPMoELayer, LocalComm  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    # forward + backward, 1-CTA and CTA-pair GEMMs, light split (E = 64 -> split active with pairs)
    for (G, E, K, d, F, T, pair) in ((4, 8, 2, 256, 256, 1024, 0), (4, 64, 4, 256, 256, 2048, 1)):
        with _lib.tuning(ffn_pair=pair):
            pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
            bias = torch.tensor(P.zipf_gate_bias(E, 1.2, 0))
            layer = P.MoELayer(pl, d, F, K, seed=1, gate_bias=bias, train=True)
            x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
            dout = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
            layer(x)
            layer.backward_step(x, dout)
            torch.cuda.synchronize()
            layer.check_status()
            print(f"layer fwd+bwd G={G} E={E} K={K} pair={pair}: ok", flush=True)
    # router tiles that cut through 64-token chunks (global atomic chunk counts)
    with _lib.tuning(router_tile_rows=80):
        pl = P.cayley_symmetric(P.ClusterShape(8, 32, 2))
        layer = P.MoELayer(pl, 256, 256, 4, seed=2, gate_bias=torch.tensor(P.zipf_gate_bias(32, 1.0, 0)))
        layer(torch.randn(2048, 256, generator=g, device="cuda").to(torch.bfloat16))
        torch.cuda.synchronize()
        layer.check_status()
        print("router tile 80: ok", flush=True)
    # router on CTA pairs (E_pad > 128), histogram zeroed in the kernel (the layer's default entry)
    with _lib.tuning(router_pair=2):
        pl = P.cayley_symmetric(P.ClusterShape(8, 256, 2))
        layer = P.MoELayer(pl, 256, 256, 8, seed=5, gate_bias=torch.tensor(P.zipf_gate_bias(256, 1.0, 0)))
        layer(torch.randn(4096, 256, generator=g, device="cuda").to(torch.bfloat16))
        torch.cuda.synchronize()
        layer.check_status()
        print("router CTA pairs E=256: ok", flush=True)
    # pipelined split on two streams
    pl = P.cayley_symmetric(P.ClusterShape(8, 16, 2))
    pip = P.MoELayer(pl, 256, 256, 2, seed=3, gate_bias=torch.tensor(P.zipf_gate_bias(16, 1.2, 1)), pipeline_ratio=0.5)
    pip(torch.randn(4096, 256, generator=g, device="cuda").to(torch.bfloat16))
    torch.cuda.synchronize()
    pip.check_status()
    print("pipelined split: ok", flush=True)
    # EP, all ranks in one process: NCCL-style exchange and NVLink peer stores
    for exchange in ("nccl", "p2p"):
        G, E, K, d, F, T = 4, 8, 2, 256, 256, 2048
        pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
        ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=4,
                        gate_bias=torch.tensor(P.zipf_gate_bias(E, 1.0, 0)), exchange=exchange)
        x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
        ep.forward([x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)])
        torch.cuda.synchronize()
        ep.check_status()
        print(f"EP LocalComm {exchange}: ok", flush=True)
    # EP pipelined split (static share exchanged on a side stream), rows regrouped per slot
    G, E, K, d, F, T = 4, 16, 2, 256, 256, 2048
    pl = P.cayley_symmetric(P.ClusterShape(G, E, 2))
    ep = EPMoELayer(pl, d, F, K, LocalComm(G), range(G), seed=6, gate_bias=torch.tensor(P.zipf_gate_bias(E, 1.0, 0)),
                    pipeline_ratio=0.5)
    x = torch.randn(T, d, generator=g, device="cuda").to(torch.bfloat16)
    ep.forward([x[r * (T // G):(r + 1) * (T // G)].contiguous() for r in range(G)])
    torch.cuda.synchronize()
    ep.check_status()
    print("EP pipelined split: ok", flush=True)
    print("sanitize run complete")


if __name__ == "__main__":
    main()
