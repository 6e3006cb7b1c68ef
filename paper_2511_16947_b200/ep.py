"""Expert-parallel MoE layer: one rank per GPU of the scheduling group.

Per micro-batch and rank r (all kernels are the sm_100a C-ABI ones):

  K1   router GEMM + top-K + this rank's histogram row      hep_gemm_bf16, hep_gate_topk
  ---  histogram all-gather -> [G][E] on every rank         comm.all_gather
  K3   identical schedule on every rank                     hep_sched_solve        (determinism, :486-487)
  K4   send positions, receive segments, split sizes        hep_moe_assign_ep
  K5   permute own tokens into the send buffer [dst][e][.]  hep_moe_permute
  ---  dispatch all-to-all-v (split sizes = pair counts)     comm.all_to_all        (router.py:181-187)
  K6   SwiGLU grouped GEMM on the received rows, local slots hep_moe_expert_ffn
  ---  combine all-to-all-v (transposed split sizes)         comm.all_to_all
  K7   weighted sum of the K returned rows per token        hep_moe_combine

Two communicators implement the two exchanges: ``DistComm`` (one process per
GPU over torch.distributed — NCCL on B200s, gloo for the CPU protocol tests)
and ``LocalComm`` (all G ranks in one process on one device, exchanges as
device copies) which lets the whole EP protocol — per-rank kernels, split
sizes, buffer layouts — run and be checked on a single GPU against the
simulated-EP ``MoELayer`` (identical bits: rows are independent in the GEMMs
and the combine sums k in a fixed order).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .core import Placement
from .layer import init_expert_weights, interleave_w13
from .scheduler import HEP_SCHED_ALL, DeviceScheduler


def _offsets(counts):
    off, acc = [], 0
    for c in counts:
        off.append(acc)
        acc += c
    return off


class LocalComm:
    """The G ranks of the group live in this process (lists indexed by rank)."""

    def __init__(self, world: int):
        self.world = world

    def all_gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        full = torch.cat(parts, dim=0)
        return [full for _ in parts]

    def all_to_all(self, sends: list[torch.Tensor], send_counts: list[list[int]],
                   recv_counts: list[list[int]]) -> list[torch.Tensor]:
        G = self.world
        offs = [_offsets(send_counts[s]) for s in range(G)]
        out = []
        for d in range(G):
            pieces = [sends[s][offs[s][d]: offs[s][d] + send_counts[s][d]] for s in range(G)]
            assert sum(p.shape[0] for p in pieces) == sum(recv_counts[d])
            out.append(torch.cat(pieces, dim=0))
        return out


class DistComm:
    """This process is one rank; collectives through torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        (p,) = parts
        chunks = [torch.empty_like(p) for _ in range(self.world)]
        self.dist.all_gather(chunks, p.contiguous(), group=self.group)
        return [torch.cat(chunks, dim=0)]

    def all_to_all(self, sends: list[torch.Tensor], send_counts: list[list[int]],
                   recv_counts: list[list[int]]) -> list[torch.Tensor]:
        (s,) = sends
        recv = torch.empty((sum(recv_counts[0]),) + tuple(s.shape[1:]), dtype=s.dtype, device=s.device)
        self.dist.all_to_all_single(recv, s, output_split_sizes=list(recv_counts[0]),
                                    input_split_sizes=list(send_counts[0]), group=self.group)
        return [recv]


class EPRank:
    """Per-rank state: local expert weights (by slot) and per-micro-batch buffers."""

    def __init__(self, layer: "EPMoELayer", rank: int, w1, w2, w3):
        self.rank = rank
        L = _lib.lib()
        dev = layer.device
        self.sched = DeviceScheduler(layer.placement, device=dev)
        nh, ns = ctypes.c_int(), ctypes.c_int()
        _lib.check(L.hep_sched_hosted(self.sched.handle, rank, ctypes.byref(nh), ctypes.byref(ns)), "hep_sched_hosted")
        self.n_hosted, self.n_slots = nh.value, max(ns.value, 1)
        F, d = layer.F, layer.d
        w13 = torch.zeros(self.n_slots, 2 * F, d, dtype=torch.bfloat16, device=dev)
        w2l = torch.zeros(self.n_slots, d, F, dtype=torch.bfloat16, device=dev)
        pl = layer.placement
        for e in pl.hosted[rank]:
            s = pl.slots[e]
            w13[s] = interleave_w13(w1[e:e + 1], w3[e:e + 1])[0]
            w2l[s] = w2[e]
        self.w13, self.w2 = w13, w2l
        self.bufs: dict[int, dict] = {}

    def buffers(self, layer: "EPMoELayer", T: int) -> dict:
        b = self.bufs.get(T)
        if b is None:
            L = _lib.lib()
            dev, K, E, G = layer.device, layer.K, layer.E, layer.G
            i32 = dict(dtype=torch.int32, device=dev)
            ws = int(L.hep_moe_assign_ep_workspace(self.sched.handle, T, K))
            n_seg = max(G * self.n_hosted, 1)
            b = dict(
                logits=torch.empty(T, layer.e_pad, dtype=torch.float32, device=dev),
                topk_idx=torch.empty(T, K, **i32),
                topk_w=torch.empty(T, K, dtype=torch.float32, device=dev),
                hist=torch.zeros(1, E, dtype=torch.int64, device=dev),
                tok_row=torch.empty(T, K, **i32),
                seg=torch.empty(n_seg, 4, **i32),
                counts=torch.empty(2 * G, dtype=torch.int64, device=dev),
                assign_ws=torch.empty(max(ws, 256), dtype=torch.uint8, device=dev),
                send=torch.empty(max(T * K, 1), layer.d, dtype=torch.bfloat16, device=dev),
                out=torch.empty(T, layer.d, dtype=torch.bfloat16, device=dev),
            )
            self.bufs[T] = b
        return b


class EPMoELayer:
    """HarmonyEP MoE layer over a real expert-parallel group.

    ``ranks`` lists the ranks this process drives: ``[comm.rank]`` with
    ``DistComm`` (one process per GPU), or ``range(G)`` with ``LocalComm``.
    Expert weights are initialised per expert id (seeded), so every replica of
    an expert is identical and the layer matches ``MoELayer``.
    """

    def __init__(self, placement: Placement, d_model: int, ffn: int, top_k: int, comm, ranks, *, seed: int = 0,
                 gate_bias: torch.Tensor | None = None, device=None):
        _lib.require_cuda()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.placement, self.comm = placement, comm
        self.G, self.E, self.K, self.d, self.F = placement.num_gpus, placement.num_experts, top_k, d_model, ffn
        if comm.world != self.G:
            raise ValueError(f"communicator has {comm.world} ranks, placement {self.G} GPUs")
        self.e_pad = max(16, (self.E + 15) // 16 * 16)
        g = torch.Generator(device=self.device).manual_seed(seed * 7919 + 17)
        wg = torch.zeros(self.e_pad, d_model, dtype=torch.bfloat16, device=self.device)
        wg[: self.E] = (torch.randn(self.E, d_model, generator=g, device=self.device) / d_model ** 0.5).to(torch.bfloat16)
        self.wg = wg
        self.gate_bias = None if gate_bias is None else gate_bias.to(self.device, torch.float32).contiguous()
        w1, w2, w3 = init_expert_weights(self.E, d_model, ffn, seed, self.device)
        self.ranks = [EPRank(self, r, w1, w2, w3) for r in ranks]
        del w1, w2, w3

    @torch.no_grad()
    def forward(self, xs: list[torch.Tensor], stream=None) -> list[torch.Tensor]:
        """xs[i] = [T][d] bf16 tokens of rank self.ranks[i]; returns their outputs."""
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            return self._forward(xs, st)

    def _forward(self, xs, st):
        L = _lib.lib()
        s = st.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        bs = []
        for rk, x in zip(self.ranks, xs):
            T = x.shape[0]
            b = rk.buffers(self, T)
            bs.append(b)
            ck(L.hep_gemm_bf16(x.data_ptr(), self.wg.data_ptr(), b["logits"].data_ptr(), T, self.e_pad, d, 0, s),
               "hep_gemm_bf16(router)")
            ck(L.hep_gate_topk(b["logits"].data_ptr(), self.e_pad, _lib.ptr(self.gate_bias), T, E, K, T, 1,
                               b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(), b["hist"].data_ptr(), s),
               "hep_gate_topk")
        hists = self.comm.all_gather([b["hist"] for b in bs])  # [G][E] on every rank
        for rk, x, b, h in zip(self.ranks, xs, bs, hists):
            T = x.shape[0]
            b["hist_all"] = h
            ck(L.hep_sched_solve(rk.sched.handle, h.data_ptr(), 1, E, None, HEP_SCHED_ALL,
                                 ctypes.byref(rk.sched.out), s), "hep_sched_solve")
            ck(L.hep_moe_assign_ep(rk.sched.handle, ctypes.byref(rk.sched.out), b["topk_idx"].data_ptr(), T, K,
                                   rk.rank, b["tok_row"].data_ptr(), b["seg"].data_ptr(), b["counts"].data_ptr(),
                                   b["assign_ws"].data_ptr(), b["assign_ws"].numel(), s), "hep_moe_assign_ep")
            ck(L.hep_moe_permute(x.data_ptr(), b["tok_row"].data_ptr(), T, K, d, b["send"].data_ptr(), s),
               "hep_moe_permute")
        # split sizes for NCCL: the only host read of the micro-batch (G x 2 integers)
        counts = [b["counts"].cpu().tolist() for b in bs]
        send_counts = [c[:G] for c in counts]
        recv_counts = [c[G:] for c in counts]
        recvs = self.comm.all_to_all([b["send"][: sum(sc)] for b, sc in zip(bs, send_counts)], send_counts,
                                     recv_counts)
        ys = []
        for rk, b, recv in zip(self.ranks, bs, recvs):
            R = recv.shape[0]
            y = torch.empty(max(R, 1), d, dtype=torch.bfloat16, device=self.device)
            if R > 0:
                h = torch.empty(R, F, dtype=torch.bfloat16, device=self.device)
                n_seg = G * rk.n_hosted
                ws = torch.empty(int(L.hep_moe_ffn_workspace(n_seg, R, rk.n_slots)), dtype=torch.uint8,
                                 device=self.device)
                ck(L.hep_moe_expert_ffn(recv.data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(), b["seg"].data_ptr(),
                                        n_seg, R, d, F, rk.n_slots, h.data_ptr(), y.data_ptr(), ws.data_ptr(),
                                        ws.numel(), rk.sched.status.data_ptr(), s), "hep_moe_expert_ffn")
            ys.append(y[:R])
        backs = self.comm.all_to_all(ys, recv_counts, send_counts)
        outs = []
        for x, b, back in zip(xs, bs, backs):
            T = x.shape[0]
            ck(L.hep_moe_combine(back.data_ptr(), b["tok_row"].data_ptr(), b["topk_w"].data_ptr(), T, K, d,
                                 b["out"].data_ptr(), s), "hep_moe_combine")
            outs.append(b["out"])
        return outs
