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

Training (``train=True``) re-lays the received rows out per local weight slot,
64-row aligned (``hep_moe_ep_train_layout`` + ``hep_moe_permute``), stores the
pre-activations, and ``backward`` runs the transposed chain with the same two
exchanges reversed, then reduces each expert's weight gradients over its EDP
group (the replicas of the expert) and the
router gradient over all ranks:

  K7^T combine backward (dY rows, dw)                       hep_moe_combine_bwd
  ---  dY all-to-all-v (dispatch split sizes)                comm.all_to_all
  K6^T SwiGLU dgrad + wgrad on the local slots               hep_moe_expert_ffn_bwd
  ---  dX all-to-all-v (combine split sizes)                 comm.all_to_all
  K1^T router backward, K5^T gather-sum into dx              hep_gate_bwd, hep_router_bwd, hep_moe_gather_sum
  ---  expert-gradient exchange inside every EDP group, router all-reduce

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
import math
from fractions import Fraction

import torch

from . import _lib
from .core import Placement, PlacementError
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

    # every driven rank's kernels run in launch order on one stream: a device-side
    # barrier between them would wait for a rank whose kernels are queued behind it
    device_sync = False

    def __init__(self, world: int):
        self.world = world

    def all_gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        full = torch.cat(parts, dim=0)
        return [full for _ in parts]

    def all_gather_int(self, v: int) -> list[int]:
        """All ranks are driven from here with the caller's (checked) shapes."""
        return [v]

    def exchange_ptrs(self, ptrs: list[int]) -> list[list[int]]:
        """Every rank's device address of a buffer, for every driven rank."""
        return [list(ptrs) for _ in ptrs]

    def barrier(self) -> None:
        """All ranks share one stream here: launch order already orders them."""

    def all_reduce(self, parts: list[torch.Tensor]) -> None:
        """In-place sum over the ranks (rank order)."""
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        for p in parts:
            p.copy_(acc)

    def all_to_all(self, sends: list[torch.Tensor], send_counts: list[list[int]],
                   recv_counts: list[list[int]], outs: list[torch.Tensor] | None = None) -> list[torch.Tensor]:
        """outs (optional): per-rank destination tensors the received rows are written into
        (their first sum(recv_counts) rows); returned in place of new tensors."""
        G = self.world
        offs = [_offsets(send_counts[s]) for s in range(G)]
        out = []
        for d in range(G):
            pieces = [sends[s][offs[s][d]: offs[s][d] + send_counts[s][d]] for s in range(G)]
            assert sum(p.shape[0] for p in pieces) == sum(recv_counts[d])
            if outs is None:
                out.append(torch.cat(pieces, dim=0))
            else:
                dst = outs[d][: sum(recv_counts[d])]
                torch.cat(pieces, dim=0, out=dst)
                out.append(dst)
        return out


class DistComm:
    """This process is one rank; collectives through torch.distributed."""

    def __init__(self, group=None, device_sync: bool = True):
        """device_sync: the NVLink exchange synchronises the ranks with device-side
        barriers / all-gathers through peer memory (hep_p2p_barrier / hep_p2p_allgather,
        no host involvement) instead of a stream drain + dist.barrier."""
        import torch.distributed as dist

        self.device_sync = device_sync
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # gloo (CPU protocol tests, or all ranks sharing one GPU): device tensors go through the host
        self.host_staged = dist.get_backend(group) == "gloo"
        self._opened: list[int] = []  # IPC mappings of peer buffers

    def _h(self, t):
        return t.cpu() if self.host_staged and t.is_cuda else t

    def all_gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        (p,) = parts
        q = self._h(p.contiguous())
        chunks = [torch.empty_like(q) for _ in range(self.world)]
        self.dist.all_gather(chunks, q, group=self.group)
        return [torch.cat(chunks, dim=0).to(p.device)]

    def all_gather_int(self, v: int) -> list[int]:
        out = [None] * self.world
        self.dist.all_gather_object(out, int(v), group=self.group)
        return out

    def exchange_ptrs(self, ptrs: list[int]) -> list[list[int]]:
        """CUDA IPC: all-gather (handle, offset) of this rank's buffer, map the peers'."""
        (ptr,) = ptrs
        L = _lib.lib()
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        _lib.check(L.hep_ipc_handle(ptr, h, ctypes.byref(off)), "hep_ipc_handle")
        allh = [None] * self.world
        self.dist.all_gather_object(allh, (bytes(h.raw), off.value), group=self.group)
        out = []
        for r, (hb, o) in enumerate(allh):
            if r == self.rank:
                out.append(ptr)
                continue
            base = ctypes.c_void_p()
            _lib.check(L.hep_ipc_open(ctypes.create_string_buffer(hb, 64), ctypes.byref(base)), "hep_ipc_open")
            self._opened.append(base.value)
            out.append(base.value + o)
        return [out]

    def barrier(self) -> None:
        """Peer writes of this rank's kernels are complete and visible once its stream
        has drained; the barrier makes every rank wait for all of them."""
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)

    def all_reduce(self, parts: list[torch.Tensor]) -> None:
        (p,) = parts
        q = self._h(p)
        self.dist.all_reduce(q, group=self.group)
        if q is not p:
            p.copy_(q)

    def all_to_all(self, sends: list[torch.Tensor], send_counts: list[list[int]],
                   recv_counts: list[list[int]], outs: list[torch.Tensor] | None = None) -> list[torch.Tensor]:
        """outs (optional): the destination tensor (its first sum(recv_counts) rows) NCCL
        receives into, instead of a new one."""
        (s,) = sends
        q = self._h(s.contiguous())
        n = sum(recv_counts[0])
        if outs is not None and not self.host_staged:
            recv = outs[0][:n]
        else:
            recv = torch.empty((n,) + tuple(s.shape[1:]), dtype=s.dtype, device=q.device)
        self.dist.all_to_all_single(recv, q, output_split_sizes=list(recv_counts[0]),
                                    input_split_sizes=list(send_counts[0]), group=self.group)
        if outs is not None and self.host_staged:
            outs[0][:n].copy_(recv)
            return [outs[0][:n]]
        return [recv.to(s.device)]


class EPRank:
    """Per-rank state: local expert weights (by slot) and per-micro-batch buffers."""

    def __init__(self, layer: "EPMoELayer", rank: int, w1=None, w2=None, w3=None, placement: Placement | None = None):
        self.rank = rank
        L = _lib.lib()
        dev = layer.device
        pl = layer.placement if placement is None else placement
        self.sched = DeviceScheduler(pl, device=dev)
        nh, ns = ctypes.c_int(), ctypes.c_int()
        _lib.check(L.hep_sched_hosted(self.sched.handle, rank, ctypes.byref(nh), ctypes.byref(ns)), "hep_sched_hosted")
        self.n_hosted, self.n_slots = nh.value, max(ns.value, 1)
        F, d = layer.F, layer.d
        self.w13 = torch.zeros(self.n_slots, 2 * F, d, dtype=torch.bfloat16, device=dev)
        self.w2 = torch.zeros(self.n_slots, d, F, dtype=torch.bfloat16, device=dev)
        if w1 is not None:
            for e in pl.hosted[rank]:
                s = pl.slots[e]
                self.w13[s] = interleave_w13(w1[e:e + 1], w3[e:e + 1])[0]
                self.w2[s] = w2[e]
        self.bufs: dict[int, dict] = {}

    def p2p_buffers(self, layer: "EPMoELayer", T: int) -> dict:
        """Exchange buffers of the NVLink path, fixed addresses (peers write into them):
        recv / h [cap][d] / [cap][F] with cap = ceil(recv_capacity_factor * T*K) rows
        (at most G*T*K, every assignment of every source), back [T*K][d] (send layout;
        peers' FFN epilogues return rows into it).  A balanced schedule delivers
        gpu_load[r] ~ T*K rows to every rank (max/mean <= 1.05 with adaptive placement);
        a micro-batch whose schedule would deliver more than cap rows to ANY rank is
        detected on the device (hep_moe_assign_ep / hep_moe_dispatch_p2p, identical
        verdict on every rank), exchanges nothing and raises CapacityError."""
        b = self.buffers(layer, T)
        if "recv" not in b:
            dev, K, G, d = layer.device, layer.K, layer.G, layer.d
            cap = max(min(G * T * K, math.ceil(layer.recv_capacity_factor * T * K)), 1)
            b["cap"] = cap
            b["recv"] = torch.empty(cap, d, dtype=torch.bfloat16, device=dev)
            b["back"] = torch.empty(max(T * K, 1), d, dtype=torch.bfloat16, device=dev)
            b["h"] = torch.empty(cap, layer.F, dtype=torch.bfloat16, device=dev)
            b["y_addr"] = torch.empty(cap, dtype=torch.int64, device=dev)
            L = _lib.lib()
            n_seg = max(G * self.n_hosted, 1)
            b["ffn_ws"] = torch.empty(max(int(L.hep_moe_ffn_workspace(n_seg, cap, self.n_slots)), 256),
                                      dtype=torch.uint8, device=dev)
            if not layer.train_mode:  # received rows regrouped per weight slot (regroup_rows)
                ns = self.n_slots
                b.update(row_map_g=torch.empty(cap, dtype=torch.int32, device=dev),
                         seg_g=torch.empty(ns, 4, dtype=torch.int32, device=dev),
                         slot_rows_g=torch.empty(ns + 1, dtype=torch.int64, device=dev),
                         rows_g=torch.empty(cap, d, dtype=torch.bfloat16, device=dev),
                         ffn_ws_g=torch.empty(max(int(L.hep_moe_ffn_workspace(ns, cap, ns)), 256), dtype=torch.uint8,
                                              device=dev))
            if layer.train_mode:  # NVLink training: the backward's two exchanges and the aligned layout
                F, ns = layer.F, self.n_slots
                Ral = cap + 63 * ns
                bf = dict(dtype=torch.bfloat16, device=dev)
                i32 = dict(dtype=torch.int32, device=dev)
                b.update(
                    dy_recv=torch.empty(cap, d, **bf),       # peers' dY rows land here (receive layout)
                    dx_back=torch.empty(max(T * K, 1), d, **bf),  # peers' dX rows return here (send layout)
                    dx_addr=torch.empty(cap, dtype=torch.int64, device=dev),
                    ident=torch.arange(max(T * K, 1), dtype=torch.int32, device=dev),
                    row_map=torch.empty(cap, **i32), seg_al=torch.empty(ns, 4, **i32),
                    slot_rows=torch.empty(ns + 1, dtype=torch.int64, device=dev), Ral=Ral,
                    rows_al=torch.zeros(Ral, d, **bf), h_al=torch.zeros(Ral, F, **bf),
                    y_al=torch.zeros(Ral, d, **bf), pre_al=torch.zeros(Ral, 2 * F, **bf),
                    ffn_ws_al=torch.empty(max(int(L.hep_moe_ffn_workspace(ns, Ral, ns)), 256), dtype=torch.uint8,
                                          device=dev))
        return b

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
                hist_buf=torch.zeros(E + (E & 1), dtype=torch.int64, device=dev),  # 16-byte rows
                router_sync=torch.zeros(4, dtype=torch.int32, device=dev),  # hep_router_topk_ws
                tok_row=torch.empty(T, K, **i32),
                seg=torch.empty(n_seg, 4, **i32),
                counts=torch.empty(2 * G, dtype=torch.int64, device=dev),
                assign_ws=torch.empty(max(ws, 256), dtype=torch.uint8, device=dev),
                send=torch.empty(max(T * K, 1), layer.d, dtype=torch.bfloat16, device=dev),
                out=torch.empty(T, layer.d, dtype=torch.bfloat16, device=dev),
            )
            b["hist"] = b["hist_buf"][:E].view(1, E)
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
                 gate_bias: torch.Tensor | None = None, device=None, train: bool = False, exchange: str = "nccl",
                 recv_capacity_factor: float = 3.0, pipeline_ratio: float | Fraction | None = None):
        """recv_capacity_factor: NVLink path receive buffers hold this many times T*K rows
        per rank (see EPRank.p2p_buffers); the NCCL path sizes its buffers per call.
        pipeline_ratio: harmony_pipelined (simulator.py:420-435, :451-453) -- the 1 - ratio
        static share of every (expert, source) is split evenly over the expert's replicas and
        dispatched (its all-to-all-v on a side stream) while the scheduled share is solved
        with the static share's GPU loads as gpu_base; NCCL exchange, forward only."""
        _lib.require_cuda()
        self.static_share = None
        if pipeline_ratio is not None:
            if not (0.0 < float(pipeline_ratio) <= 1.0):
                raise ValueError("pipeline_ratio must be in (0, 1]")  # SimulationConfig (simulator.py:117-118)
            if train or exchange != "nccl":
                raise ValueError("the pipelined split runs on the NCCL exchange, forward only")
            self.static_share = Fraction(1) - Fraction(pipeline_ratio)
            self._side = torch.cuda.Stream()
        if recv_capacity_factor <= 0:
            raise ValueError("recv_capacity_factor must be positive")
        self.recv_capacity_factor = float(recv_capacity_factor)
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' (all-to-all-v collectives) or 'p2p' (NVLink peer stores)")
        self.exchange = exchange
        self._peer_tables: dict[int, list] = {}
        self._peer_tables_bwd: dict[int, list] = {}
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.placement, self.comm = placement, comm
        self.G, self.E, self.K, self.d, self.F = placement.num_gpus, placement.num_experts, top_k, d_model, ffn
        if comm.world != self.G:
            raise ValueError(f"communicator has {comm.world} ranks, placement {self.G} GPUs")
        self.train_mode = train
        self.e_pad = max(16, (self.E + 15) // 16 * 16)
        self.e64 = (self.E + 63) // 64 * 64  # router rows padded to 64 for its backward GEMMs
        g = torch.Generator(device=self.device).manual_seed(seed * 7919 + 17)
        wg = torch.zeros(self.e64, d_model, dtype=torch.bfloat16, device=self.device)
        wg[: self.E] = (torch.randn(self.E, d_model, generator=g, device=self.device) / d_model ** 0.5).to(torch.bfloat16)
        self.wg = wg
        self.gate_bias = None if gate_bias is None else gate_bias.to(self.device, torch.float32).contiguous()
        w1, w2, w3 = init_expert_weights(self.E, d_model, ffn, seed, self.device)
        self.ranks = [EPRank(self, r, w1, w2, w3) for r in ranks]
        del w1, w2, w3
        # inference: regroup the received rows per local weight slot before the FFN (NCCL path:
        # _ffn_rows; NVLink path: the return addresses move with the rows); False runs the FFN
        # on the [src][expert] runs directly
        self.regroup_rows = True

    @torch.no_grad()
    def migrate(self, placement: Placement) -> dict:
        """Adopt a new placement (adaptive replacement, ``adaptive.py:119-166``) by moving
        expert weights between GPUs: every replica the new placement adds on a GPU is
        fetched from the lowest-id GPU that held the expert before (one all-to-all-v of
        weight panels), replicas that stay on a GPU are copied between local slots.
        Returns the moved-replica count (= the reference's ``changed_slots``, the
        (expert, GPU) pairs new to the placement) and this process's bytes sent."""
        if (placement.num_gpus, placement.num_experts) != (self.G, self.E):
            raise ValueError("placement must keep the number of GPUs and experts")
        new_ranks = [EPRank(self, rk.rank, placement=placement) for rk in self.ranks]
        stats = migrate_weights(self.placement, placement, self.comm, [rk.rank for rk in self.ranks],
                                [rk.w13 for rk in self.ranks], [rk.w2 for rk in self.ranks],
                                [nr.w13 for nr in new_ranks], [nr.w2 for nr in new_ranks])
        self.placement = placement
        self.ranks = new_ranks
        self._peer_tables.clear()  # new exchange buffers: peers re-map them on the next forward
        self._peer_tables_bwd.clear()
        return stats

    @torch.no_grad()
    def forward(self, xs: list[torch.Tensor], stream=None, events: dict | None = None) -> list[torch.Tensor]:
        """xs[i] = [T][d] bf16 tokens of rank self.ranks[i]; returns their outputs.
        ``events`` optionally maps "ffn" (the expert FFN launches) and "a2a" (the dispatch
        exchange: the peer-store dispatch kernel, or the NCCL all-to-all-v) to a
        (start, end) torch.cuda.Event pair."""
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            if self.exchange == "p2p":
                return self._forward_p2p(xs, st, events or {})
            if self.static_share is not None:
                return self._forward_pipelined(xs, st, events or {})
            return self._forward(xs, st, events or {})

    def _peer_table(self, T: int) -> list:
        """Per driven rank: device tables of every rank's receive / return buffer address.
        Building it is collective; it also checks that every rank has the same T (the
        peer buffers' capacities and the peers' store addresses assume it)."""
        tab = self._peer_tables.get(T)
        if tab is None:
            all_t = self.comm.all_gather_int(T) if hasattr(self.comm, "all_gather_int") else [T]
            if any(t != T for t in all_t):
                raise ValueError(f"the NVLink exchange needs the same token count on every rank, got {all_t}")
            bs = [rk.p2p_buffers(self, T) for rk in self.ranks]
            recv = self.comm.exchange_ptrs([b["recv"].data_ptr() for b in bs])
            back = self.comm.exchange_ptrs([b["back"].data_ptr() for b in bs])
            tab = [(torch.tensor(rv, dtype=torch.int64, device=self.device),
                    torch.tensor(bk, dtype=torch.int64, device=self.device)) for rv, bk in zip(recv, back)]
            if self.train_mode:
                dyr = self.comm.exchange_ptrs([b["dy_recv"].data_ptr() for b in bs])
                dxb = self.comm.exchange_ptrs([b["dx_back"].data_ptr() for b in bs])
                self._peer_tables_bwd[T] = [(torch.tensor(a, dtype=torch.int64, device=self.device),
                                             torch.tensor(c, dtype=torch.int64, device=self.device))
                                            for a, c in zip(dyr, dxb)]
            self._peer_tables[T] = tab
        return tab

    def _sync_table(self) -> list:
        """Device-side synchronisation state per driven rank (built once): flags [G + 2]
        uint32 (arrival epochs, own epoch counter, timeout flag) and the gathered histogram
        hist_all [G][E2] int64, both mapped by every peer, with device tables of the
        peers' addresses."""
        if getattr(self, "_sync", None) is None:
            G, E2 = self.G, self.E + (self.E & 1)
            flags = [torch.zeros(G + 2, dtype=torch.int32, device=self.device) for _ in self.ranks]
            hall = [torch.zeros(G, E2, dtype=torch.int64, device=self.device) for _ in self.ranks]
            pf = self.comm.exchange_ptrs([f.data_ptr() for f in flags])
            ph = self.comm.exchange_ptrs([h.data_ptr() for h in hall])
            self._sync = [(f, h, torch.tensor(a, dtype=torch.int64, device=self.device),
                           torch.tensor(b, dtype=torch.int64, device=self.device))
                          for f, h, a, b in zip(flags, hall, pf, ph)]
        return self._sync

    def check_status(self) -> None:
        """Raise the reference exception class for a device-detected error of the last
        micro-batch on any driven rank (scheduler, assignment, receive capacity)."""
        for rk in self.ranks:
            rk.sched.check_status(f"EPMoELayer rank {rk.rank}")

    def check_sync(self) -> None:
        """Raise if a device-side barrier of this layer gave up waiting for a peer."""
        for flags, _, _, _ in getattr(self, "_sync", None) or []:
            if int(flags[self.G + 1].item()):
                raise RuntimeError("EP device barrier timed out: a peer rank never arrived")

    def _device_barrier(self, s) -> None:
        L = _lib.lib()
        for rk, (flags, _, pflags, _) in zip(self.ranks, self._sync_table()):
            _lib.check(L.hep_p2p_barrier(pflags.data_ptr(), flags.data_ptr(), rk.rank, self.G, s), "hep_p2p_barrier")

    def _forward_p2p(self, xs, st, ev):
        """Forward with both exchanges as NVLink peer stores: the dispatch kernel writes
        rows into the destination ranks' receive buffers, the down-projection GEMM's
        epilogue writes expert outputs into the source ranks' return buffers.  The only
        collectives are the histogram all-gather and two barriers (no host reads of the
        schedule, no NCCL on the data path)."""
        L = _lib.lib()
        s = st.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        T0 = xs[0].shape[0]
        if any(x.shape[0] != T0 for x in xs):
            raise ValueError("the NVLink exchange needs the same token count on every rank "
                             f"(got {[x.shape[0] for x in xs]})")
        tabs = self._peer_table(T0)
        bs = []
        for rk, x in zip(self.ranks, xs):
            T = x.shape[0]
            b = rk.p2p_buffers(self, T)
            bs.append(b)
            ck(L.hep_router_topk_ws(x.data_ptr(), self.wg.data_ptr(), T, d, E, self.e_pad, _lib.ptr(self.gate_bias), K,
                                    T, 1, b["logits"].data_ptr(), b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(),
                                    b["hist"].data_ptr(), None, b["router_sync"].data_ptr(), s), "hep_router_topk")
        sync = getattr(self.comm, "device_sync", False)
        if sync:  # histogram rows straight into every peer's hist_all, then a device barrier
            E2 = E + (E & 1)
            hists = []
            for rk, b, (flags, hall, pflags, phall) in zip(self.ranks, bs, self._sync_table()):
                ck(L.hep_p2p_allgather(b["hist_buf"].data_ptr(), 8 * E2, phall.data_ptr(), pflags.data_ptr(),
                                       flags.data_ptr(), rk.rank, G, s), "hep_p2p_allgather")
                hists.append(hall)
            hist_stride = E2
        else:
            hists = self.comm.all_gather([b["hist"] for b in bs])
            hist_stride = E
        for rk, x, b, h, (p_recv, p_back) in zip(self.ranks, xs, bs, hists, tabs):
            T = x.shape[0]
            b["hist_all"] = h[:, :E]  # [G][E] view (device-gathered rows are padded to even E)
            ck(L.hep_sched_solve(rk.sched.handle, h.data_ptr(), 1, hist_stride, None, HEP_SCHED_ALL,
                                 ctypes.byref(rk.sched.out), s), "hep_sched_solve")
            ck(L.hep_moe_assign_ep(rk.sched.handle, ctypes.byref(rk.sched.out), b["topk_idx"].data_ptr(), T, K,
                                   rk.rank, b["cap"], b["tok_row"].data_ptr(), b["seg"].data_ptr(),
                                   b["counts"].data_ptr(), b["assign_ws"].data_ptr(), b["assign_ws"].numel(), s),
               "hep_moe_assign_ep")
            if "a2a" in ev:
                ev["a2a"][0].record(st)
            ck(L.hep_moe_dispatch_p2p(x.data_ptr(), b["tok_row"].data_ptr(), T, K, d, rk.rank, G,
                                      rk.sched.transfer.data_ptr(), p_recv.data_ptr(), b["cap"],
                                      rk.sched.status.data_ptr(), s), "hep_moe_dispatch_p2p")
            if "a2a" in ev:
                ev["a2a"][1].record(st)
            if self.regroup_rows and not self.train_mode:  # regrouped: rows per weight slot, return addresses with them
                ck(L.hep_moe_ep_train_layout(b["seg"].data_ptr(), rk.n_hosted, G, rk.n_slots, 1,
                                             b["row_map_g"].data_ptr(), b["cap"], b["seg_g"].data_ptr(),
                                             b["slot_rows_g"].data_ptr(), s), "hep_moe_ep_train_layout")
                ck(L.hep_moe_return_addr_map(rk.sched.transfer.data_ptr(), rk.rank, G, p_back.data_ptr(), d * 2,
                                             b["cap"], b["row_map_g"].data_ptr(), b["y_addr"].data_ptr(), s),
                   "hep_moe_return_addr_map")
            else:
                ck(L.hep_moe_return_addr(rk.sched.transfer.data_ptr(), rk.rank, G, p_back.data_ptr(), d * 2, b["cap"],
                                         b["y_addr"].data_ptr(), s), "hep_moe_return_addr")
        if sync:
            self._device_barrier(s)  # every receive buffer complete
        else:
            self.comm.barrier()
        if "ffn" in ev:
            ev["ffn"][0].record(st)
        for rk, b, x in zip(self.ranks, bs, xs):
            n_seg = G * rk.n_hosted
            x_rows = x.shape[0]  # balanced schedule: about T*K rows land on every rank
            if self.train_mode:
                self._train_ffn_p2p(rk, b, s)
                b["x"] = x
                continue
            if n_seg and self.regroup_rows:  # one run per weight slot; outputs still go straight to the sources
                ck(L.hep_moe_permute(b["recv"].data_ptr(), b["row_map_g"].data_ptr(), b["cap"], 1, d,
                                     b["rows_g"].data_ptr(), s), "hep_moe_permute(regroup)")
                ck(L.hep_moe_expert_ffn_p2p(b["rows_g"].data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(),
                                            b["seg_g"].data_ptr(), rk.n_slots, b["cap"], x_rows * K, d, F, rk.n_slots,
                                            b["h"].data_ptr(), b["y_addr"].data_ptr(), b["ffn_ws_g"].data_ptr(),
                                            b["ffn_ws_g"].numel(), rk.sched.status.data_ptr(), s),
                   "hep_moe_expert_ffn_p2p")
            elif n_seg:
                ck(L.hep_moe_expert_ffn_p2p(b["recv"].data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(),
                                            b["seg"].data_ptr(), n_seg, b["cap"], x_rows * K, d, F, rk.n_slots,
                                            b["h"].data_ptr(),
                                            b["y_addr"].data_ptr(), b["ffn_ws"].data_ptr(), b["ffn_ws"].numel(),
                                            rk.sched.status.data_ptr(), s), "hep_moe_expert_ffn_p2p")
        if "ffn" in ev:
            ev["ffn"][1].record(st)
        if sync:
            self._device_barrier(s)  # every expert output back at its source
        else:
            self.comm.barrier()
        outs = []
        for x, b in zip(xs, bs):
            T = x.shape[0]
            ck(L.hep_moe_combine(b["back"].data_ptr(), b["tok_row"].data_ptr(), b["topk_w"].data_ptr(), T, K, d,
                                 b["out"].data_ptr(), s), "hep_moe_combine")
            outs.append(b["out"])
        return outs

    def _train_ffn_p2p(self, rk: EPRank, b: dict, s) -> None:
        """NVLink training forward, FFN part: the received rows (count known only on the
        device) are laid out per local weight slot, 64-row aligned (row_map entries past the
        count are -1 and skipped), the training FFN keeps the pre-activations, and the output
        rows go straight back into the sources' return buffers."""
        L = _lib.lib()
        ck = _lib.check
        G, d, F = self.G, self.d, self.F
        ns, cap, Ral = rk.n_slots, b["cap"], b["Ral"]
        st = rk.sched.status.data_ptr()
        ck(L.hep_moe_ep_train_layout(b["seg"].data_ptr(), rk.n_hosted, G, ns, 64, b["row_map"].data_ptr(), cap,
                                     b["seg_al"].data_ptr(), b["slot_rows"].data_ptr(), s), "hep_moe_ep_train_layout")
        ck(L.hep_moe_permute(b["recv"].data_ptr(), b["row_map"].data_ptr(), cap, 1, d, b["rows_al"].data_ptr(), s),
           "hep_moe_permute(align)")
        # padding rows are never written by the GEMMs, the weight-gradient GEMMs contract over
        # them: X and H padding must be zero
        ck(L.hep_moe_zero_padding(b["slot_rows"].data_ptr(), b["seg_al"].data_ptr(), ns, ns, b["rows_al"].data_ptr(), d,
                                  s), "hep_moe_zero_padding(rows)")
        ck(L.hep_moe_zero_padding(b["slot_rows"].data_ptr(), b["seg_al"].data_ptr(), ns, ns, b["h_al"].data_ptr(), F,
                                  s), "hep_moe_zero_padding(h)")
        ck(L.hep_moe_expert_ffn_train(b["rows_al"].data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(),
                                      b["seg_al"].data_ptr(), ns, Ral, d, F, ns, b["h_al"].data_ptr(),
                                      b["y_al"].data_ptr(), b["pre_al"].data_ptr(), b["ffn_ws_al"].data_ptr(),
                                      b["ffn_ws_al"].numel(), st, s), "hep_moe_expert_ffn_train")
        ck(L.hep_moe_rows_to_addr(b["y_al"].data_ptr(), b["row_map"].data_ptr(), rk.sched.transfer.data_ptr(), rk.rank,
                                  G, cap, d, b["y_addr"].data_ptr(), st, s), "hep_moe_rows_to_addr(y)")

    def _backward_p2p(self, douts, st):
        """NVLink training backward: dY rows stored into the destinations' receive buffers
        (the dispatch kernel on the send layout), the expert FFN backward on the aligned
        layout, dX rows stored back into the sources' buffers, device barriers between."""
        L = _lib.lib()
        s = st.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        dev = self.device
        T = douts[0].shape[0]
        bs = [rk.p2p_buffers(self, T) for rk in self.ranks]
        tabs = self._peer_table(T)
        btabs = self._peer_tables_bwd[T]
        dws = []
        for rk, b, dout, (p_recv, p_back), (p_dyrecv, p_dxback) in zip(self.ranks, bs, douts, tabs, btabs):
            dy = torch.empty(max(T * K, 1), d, dtype=torch.bfloat16, device=dev)
            dw = torch.empty(T, K, dtype=torch.float32, device=dev)
            ck(L.hep_moe_combine_bwd(dout.contiguous().data_ptr(), b["back"].data_ptr(), b["tok_row"].data_ptr(),
                                     b["topk_w"].data_ptr(), T, K, d, dy.data_ptr(), dw.data_ptr(), s),
               "hep_moe_combine_bwd")
            # every send position p (= its row of dy) to its destination's receive slot
            ck(L.hep_moe_dispatch_p2p(dy.data_ptr(), b["ident"].data_ptr(), T * K, 1, d, rk.rank, G,
                                      rk.sched.transfer.data_ptr(), p_dyrecv.data_ptr(), b["cap"],
                                      rk.sched.status.data_ptr(), s), "hep_moe_dispatch_p2p(dY)")
            ck(L.hep_moe_return_addr(rk.sched.transfer.data_ptr(), rk.rank, G, p_dxback.data_ptr(), d * 2, b["cap"],
                                     b["dx_addr"].data_ptr(), s), "hep_moe_return_addr(dX)")
            b["dy_keep"] = dy
            dws.append(dw)
        self._sync_ranks(s)  # every dY row arrived
        dw13s, dw2s = [], []
        for rk, b in zip(self.ranks, bs):
            ns, Ral, cap = rk.n_slots, b["Ral"], b["cap"]
            bf = dict(dtype=torch.bfloat16, device=dev)
            dy_al = torch.zeros(Ral, d, **bf)
            ck(L.hep_moe_permute(b["dy_recv"].data_ptr(), b["row_map"].data_ptr(), cap, 1, d, dy_al.data_ptr(), s),
               "hep_moe_permute(dY align)")
            da13 = torch.empty(Ral, 2 * F, **bf)
            dx_al = torch.empty(Ral, d, **bf)
            dw13 = torch.empty(ns, 2 * F, d, dtype=torch.float32, device=dev)
            dw2 = torch.empty(ns, d, F, dtype=torch.float32, device=dev)
            ck(L.hep_moe_expert_ffn_bwd(b["rows_al"].data_ptr(), b["pre_al"].data_ptr(), b["h_al"].data_ptr(),
                                        dy_al.data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(), b["seg_al"].data_ptr(),
                                        ns, b["slot_rows"].data_ptr(), Ral, d, F, ns, da13.data_ptr(),
                                        dx_al.data_ptr(), dw13.data_ptr(), dw2.data_ptr(), b["ffn_ws_al"].data_ptr(),
                                        b["ffn_ws_al"].numel(), rk.sched.status.data_ptr(), s),
               "hep_moe_expert_ffn_bwd")
            ck(L.hep_moe_rows_to_addr(dx_al.data_ptr(), b["row_map"].data_ptr(), rk.sched.transfer.data_ptr(),
                                      rk.rank, G, cap, d, b["dx_addr"].data_ptr(), rk.sched.status.data_ptr(), s),
               "hep_moe_rows_to_addr(dX)")
            b["dx_al_keep"] = dx_al
            dw13s.append(dw13)
            dw2s.append(dw2)
        self._sync_ranks(s)  # every dX row is back at its source
        dxs, dwgs = [], []
        for b, dw in zip(bs, dws):
            x = b["x"]
            dlogits = torch.empty(T, self.e64, dtype=torch.bfloat16, device=dev)
            dwg = torch.empty(self.e64, d, dtype=torch.float32, device=dev)
            dxg = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            dx = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            ck(L.hep_gate_bwd(b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(), dw.data_ptr(), T, K, self.e64,
                              dlogits.data_ptr(), s), "hep_gate_bwd")
            ck(L.hep_router_bwd(x.data_ptr(), self.wg.data_ptr(), dlogits.data_ptr(), T, d, self.e64,
                                dwg.data_ptr(), dxg.data_ptr(), s), "hep_router_bwd")
            ck(L.hep_moe_gather_sum(b["dx_back"].data_ptr(), b["tok_row"].data_ptr(), None, dxg.data_ptr(), T, K, d,
                                    dx.data_ptr(), s), "hep_moe_gather_sum")
            dxs.append(dx)
            dwgs.append(dwg)
        self.comm.all_reduce(dwgs)
        edp_reduce(self.placement, self.comm, [rk.rank for rk in self.ranks], dw13s, dw2s)
        return [(dx, dwg[:E], dw13, dw2) for dx, dwg, dw13, dw2 in zip(dxs, dwgs, dw13s, dw2s)]

    def _sync_ranks(self, s) -> None:
        """Order the exchanges across ranks: device barrier (DistComm device_sync) or a
        stream drain + host barrier."""
        if getattr(self.comm, "device_sync", False):
            self._device_barrier(s)
        else:
            self.comm.barrier()

    def _forward(self, xs, st, ev):
        L = _lib.lib()
        s = st.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        bs = []
        for rk, x in zip(self.ranks, xs):
            T = x.shape[0]
            b = rk.buffers(self, T)
            bs.append(b)
            ck(L.hep_router_topk_ws(x.data_ptr(), self.wg.data_ptr(), T, d, E, self.e_pad, _lib.ptr(self.gate_bias), K,
                                    T, 1, b["logits"].data_ptr(), b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(),
                                    b["hist"].data_ptr(), None, b["router_sync"].data_ptr(), s), "hep_router_topk")
        hists = self.comm.all_gather([b["hist"] for b in bs])  # [G][E] on every rank
        for rk, x, b, h in zip(self.ranks, xs, bs, hists):
            T = x.shape[0]
            b["hist_all"] = h
            ck(L.hep_sched_solve(rk.sched.handle, h.data_ptr(), 1, E, None, HEP_SCHED_ALL,
                                 ctypes.byref(rk.sched.out), s), "hep_sched_solve")
            ck(L.hep_moe_assign_ep(rk.sched.handle, ctypes.byref(rk.sched.out), b["topk_idx"].data_ptr(), T, K,
                                   rk.rank, 0, b["tok_row"].data_ptr(), b["seg"].data_ptr(), b["counts"].data_ptr(),
                                   b["assign_ws"].data_ptr(), b["assign_ws"].numel(), s), "hep_moe_assign_ep")
            ck(L.hep_moe_permute(x.data_ptr(), b["tok_row"].data_ptr(), T, K, d, b["send"].data_ptr(), s),
               "hep_moe_permute")
        # split sizes for NCCL: the only host read of the micro-batch (G x 2 integers)
        counts = [b["counts"].cpu().tolist() for b in bs]
        send_counts = [c[:G] for c in counts]
        recv_counts = [c[G:] for c in counts]
        if "a2a" in ev:
            ev["a2a"][0].record(st)
        recvs = self.comm.all_to_all([b["send"][: sum(sc)] for b, sc in zip(bs, send_counts)], send_counts,
                                     recv_counts)
        if "a2a" in ev:
            ev["a2a"][1].record(st)
        ys = []
        if "ffn" in ev:
            ev["ffn"][0].record(st)
        for rk, b, recv in zip(self.ranks, bs, recvs):
            b["R_recv"] = recv.shape[0]
            ys.append(self._expert_ffn(rk, b, recv))
        if "ffn" in ev:
            ev["ffn"][1].record(st)
        for i, b in enumerate(bs):
            b["send_counts"], b["recv_counts"] = send_counts[i], recv_counts[i]
        backs = self.comm.all_to_all(ys, recv_counts, send_counts)
        outs = []
        for x, b, back in zip(xs, bs, backs):
            T = x.shape[0]
            if self.train_mode:
                b["x"], b["back"] = x, back
            ck(L.hep_moe_combine(back.data_ptr(), b["tok_row"].data_ptr(), b["topk_w"].data_ptr(), T, K, d,
                                 b["out"].data_ptr(), s), "hep_moe_combine")
            outs.append(b["out"])
        return outs

    def _phase_buffers(self, rk: EPRank, T: int) -> dict:
        """Per-rank buffers of the pipelined split: the phases' row maps, segments, split
        sizes and workspaces (they run on two streams), one send buffer holding phase 0's
        rows at [0, T*K) and phase 1's at [T*K, 2*T*K)."""
        b = rk.buffers(self, T)
        if "send2" not in b:
            L = _lib.lib()
            dev, K, G = self.device, self.K, self.G
            i32 = dict(dtype=torch.int32, device=dev)
            ws = max(int(L.hep_moe_assign_ep_workspace(rk.sched.handle, T, K)), 256)
            n_seg = max(G * rk.n_hosted, 1)
            b.update(
                tok_row_ph=[torch.empty(T, K, **i32) for _ in range(2)],
                seg_ph=[torch.empty(n_seg, 4, **i32) for _ in range(2)],
                counts_ph=[torch.empty(2 * G, dtype=torch.int64, device=dev) for _ in range(2)],
                assign_ws_ph=[torch.empty(ws, dtype=torch.uint8, device=dev) for _ in range(2)],
                send2=torch.empty(max(2 * T * K, 1), self.d, dtype=torch.bfloat16, device=dev),
                # both phases' received rows; at most every source's T*K assignments
                recv2=torch.empty(max(G * T * K, 1), self.d, dtype=torch.bfloat16, device=dev),
                back2=torch.zeros(max(2 * T * K, 1), self.d, dtype=torch.bfloat16, device=dev),
            )
        return b

    def _forward_pipelined(self, xs, st, ev):
        """harmony_pipelined over the EP group (simulator.py:420-435, :451-453).  Per rank:
        router -> histogram all-gather -> hep_sched_pipelined (split; the static phase's
        even plan, routing and transfer plan on the side stream; the scheduled share's
        solve with gpu_base on this stream).  The static phase's assignment, permute and
        all-to-all-v run on the side stream (the host reads only its split sizes) while
        the scheduled phase is solved, assigned and exchanged here; the expert FFN then
        runs once over both phases' received rows (one weight stream), the outputs go
        back per phase, and the combine reads both phases' returned rows."""
        L = _lib.lib()
        s = st.cuda_stream
        side = self._side
        ss = side.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        bs = []
        for rk, x in zip(self.ranks, xs):
            T = x.shape[0]
            b = self._phase_buffers(rk, T)
            bs.append(b)
            ck(L.hep_router_topk_ws(x.data_ptr(), self.wg.data_ptr(), T, d, E, self.e_pad, _lib.ptr(self.gate_bias), K,
                                    T, 1, b["logits"].data_ptr(), b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(),
                                    b["hist"].data_ptr(), None, b["router_sync"].data_ptr(), s), "hep_router_topk")
        hists = self.comm.all_gather([b["hist"] for b in bs])  # [G][E] on every rank
        for rk, x, b, h in zip(self.ranks, xs, bs, hists):
            T = x.shape[0]
            b["hist_all"] = h
            rk.sched.launch_pipelined(h, 1, E, self.static_share, HEP_SCHED_ALL, st, stream_static=side)
            split = rk.sched.split.data_ptr()
            # phase 0 (static share) on the side stream, behind its plan
            ck(L.hep_moe_assign_ep_phase(rk.sched.handle, ctypes.byref(rk.sched.former.out), split, 0,
                                         b["topk_idx"].data_ptr(), T, K, rk.rank, 0, b["tok_row"].data_ptr(),
                                         b["tok_row_ph"][0].data_ptr(), b["seg_ph"][0].data_ptr(),
                                         b["counts_ph"][0].data_ptr(), b["assign_ws_ph"][0].data_ptr(),
                                         b["assign_ws_ph"][0].numel(), ss), "hep_moe_assign_ep_phase(static)")
            ck(L.hep_moe_permute(x.data_ptr(), b["tok_row_ph"][0].data_ptr(), T, K, d, b["send2"].data_ptr(), ss),
               "hep_moe_permute(static)")
        with torch.cuda.stream(side):
            # the static share's split sizes (a side-stream sync: the solve keeps running)
            c0 = [b["counts_ph"][0].cpu().tolist() for b in bs]
            recv0 = self.comm.all_to_all([b["send2"][: sum(c[:G])] for b, c in zip(bs, c0)], [c[:G] for c in c0],
                                         [c[G:] for c in c0], outs=[b["recv2"] for b in bs])
        for rk, x, b in zip(self.ranks, xs, bs):
            T = x.shape[0]
            ck(L.hep_moe_assign_ep_phase(rk.sched.handle, ctypes.byref(rk.sched.out), rk.sched.split.data_ptr(), 1,
                                         b["topk_idx"].data_ptr(), T, K, rk.rank, T * K, b["tok_row"].data_ptr(),
                                         b["tok_row_ph"][1].data_ptr(), b["seg_ph"][1].data_ptr(),
                                         b["counts_ph"][1].data_ptr(), b["assign_ws_ph"][1].data_ptr(),
                                         b["assign_ws_ph"][1].numel(), s), "hep_moe_assign_ep_phase(scheduled)")
            ck(L.hep_moe_permute(x.data_ptr(), b["tok_row_ph"][1].data_ptr(), T, K, d, b["send2"].data_ptr(), s),
               "hep_moe_permute(scheduled)")
        c1 = [b["counts_ph"][1].cpu().tolist() for b in bs]
        if "a2a" in ev:
            ev["a2a"][0].record(st)
        # phase 1's rows land right after phase 0's in the same receive buffer (no concatenation)
        recv1 = self.comm.all_to_all([b["send2"][x.shape[0] * K: x.shape[0] * K + sum(c[:G])]
                                      for b, c, x in zip(bs, c1, xs)], [c[:G] for c in c1], [c[G:] for c in c1],
                                     outs=[b["recv2"][sum(a[G:]):] for b, a in zip(bs, c0)])
        if "a2a" in ev:
            ev["a2a"][1].record(st)
        st.wait_stream(side)
        ys0, ys1 = [], []
        if "ffn" in ev:
            ev["ffn"][0].record(st)
        for rk, b, r0, r1 in zip(self.ranks, bs, recv0, recv1):
            R0, R1 = r0.shape[0], r1.shape[0]
            recv = b["recv2"][: R0 + R1]  # [phase 0 rows | phase 1 rows]
            seg1 = b["seg_ph"][1].clone()
            seg1[:, 0] += R0  # phase 1's rows follow phase 0's in the FFN input
            seg = torch.cat([b["seg_ph"][0], seg1], dim=0)
            y = torch.empty(max(R0 + R1, 1), d, dtype=torch.bfloat16, device=self.device)
            if R0 + R1 > 0:  # 2G source blocks: [phase][src][hosted expert]
                self._ffn_rows(rk, recv, seg, 2 * G, y)
            ys0.append(y[:R0])
            ys1.append(y[R0:R0 + R1])
        if "ffn" in ev:
            ev["ffn"][1].record(st)
        # the outputs return straight to their send positions (phase 1's from T*K on)
        self.comm.all_to_all(ys0, [c[G:] for c in c0], [c[:G] for c in c0], outs=[b["back2"] for b in bs])
        self.comm.all_to_all(ys1, [c[G:] for c in c1], [c[:G] for c in c1],
                             outs=[b["back2"][x.shape[0] * K:] for b, x in zip(bs, xs)])
        outs = []
        for x, b, a, c in zip(xs, bs, c0, c1):
            T = x.shape[0]
            back = b["back2"]
            b["send_counts_ph"], b["recv_counts_ph"] = [a[:G], c[:G]], [a[G:], c[G:]]
            b["R_recv"] = sum(a[G:]) + sum(c[G:])
            ck(L.hep_moe_combine(back.data_ptr(), b["tok_row"].data_ptr(), b["topk_w"].data_ptr(), T, K, d,
                                 b["out"].data_ptr(), s), "hep_moe_combine")
            outs.append(b["out"])
        return outs

    def _ffn_rows(self, rk: EPRank, recv: torch.Tensor, seg: torch.Tensor, n_blocks: int, y: torch.Tensor) -> None:
        """K6 over received rows in the all-to-all-v layout ([src][hosted expert]: n_blocks
        source blocks, seg [n_blocks * n_hosted][4]); Y into y in the same order.  With
        regroup_rows the rows are first gathered into one contiguous run per local weight
        slot (hep_moe_ep_train_layout with row_align 1, a permute), so an expert's rows
        from all sources share m-tiles instead of each (source, expert) run filling its
        own partial tiles, and the outputs are gathered back afterwards."""
        L = _lib.lib()
        ck = _lib.check
        s = torch.cuda.current_stream().cuda_stream
        d, F, ns = self.d, self.F, rk.n_slots
        R = recv.shape[0]
        dev = self.device
        if self.regroup_rows:
            i32 = dict(dtype=torch.int32, device=dev)
            row_map = torch.empty(R, **i32)
            seg_al = torch.empty(ns, 4, **i32)
            slot_rows = torch.empty(ns + 1, dtype=torch.int64, device=dev)
            ck(L.hep_moe_ep_train_layout(seg.data_ptr(), rk.n_hosted, n_blocks, ns, 1, row_map.data_ptr(), 0,
                                         seg_al.data_ptr(), slot_rows.data_ptr(), s), "hep_moe_ep_train_layout")
            rows = torch.empty(R, d, dtype=torch.bfloat16, device=dev)
            ck(L.hep_moe_permute(recv.data_ptr(), row_map.data_ptr(), R, 1, d, rows.data_ptr(), s),
               "hep_moe_permute(regroup)")
            src_rows, src_seg, n_seg, y_out = rows, seg_al, ns, torch.empty(R, d, dtype=torch.bfloat16, device=dev)
        else:
            src_rows, src_seg, n_seg, y_out = recv, seg, n_blocks * rk.n_hosted, y
        h = torch.empty(R, F, dtype=torch.bfloat16, device=dev)
        ws = torch.empty(int(L.hep_moe_ffn_workspace(n_seg, R, ns)), dtype=torch.uint8, device=dev)
        ck(L.hep_moe_expert_ffn(src_rows.data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(), src_seg.data_ptr(), n_seg, R,
                                d, F, ns, h.data_ptr(), y_out.data_ptr(), ws.data_ptr(), ws.numel(),
                                rk.sched.status.data_ptr(), s), "hep_moe_expert_ffn")
        if self.regroup_rows:  # back to the receive order
            ck(L.hep_moe_gather_sum(y_out.data_ptr(), row_map.data_ptr(), None, None, R, 1, d, y.data_ptr(), s),
               "hep_moe_gather_sum(ungroup)")

    def _expert_ffn(self, rk: EPRank, b: dict, recv: torch.Tensor) -> torch.Tensor:
        """K6 on the received rows of one rank; returns Y in receive order."""
        L = _lib.lib()
        ck = _lib.check
        s = torch.cuda.current_stream().cuda_stream
        G, d, F = self.G, self.d, self.F
        R = recv.shape[0]
        y = torch.empty(max(R, 1), d, dtype=torch.bfloat16, device=self.device)
        if not self.train_mode:
            if R > 0:
                self._ffn_rows(rk, recv, b["seg"], G, y)
            return y[:R]
        # training: per-slot 64-row aligned blocks (weight-gradient GEMMs), pre-activations kept
        ns = rk.n_slots
        i32 = dict(dtype=torch.int32, device=self.device)
        row_map = torch.empty(max(R, 1), **i32)
        seg_al = torch.empty(ns, 4, **i32)
        slot_rows = torch.empty(ns + 1, dtype=torch.int64, device=self.device)
        ck(L.hep_moe_ep_train_layout(b["seg"].data_ptr(), rk.n_hosted, G, ns, 64, row_map.data_ptr(), 0,
                                     seg_al.data_ptr(), slot_rows.data_ptr(), s), "hep_moe_ep_train_layout")
        Ral = R + 63 * ns
        bf = dict(dtype=torch.bfloat16, device=self.device)
        rows_al = torch.empty(max(Ral, 1), d, **bf)
        h_al = torch.empty(max(Ral, 1), F, **bf)
        y_al = torch.empty(max(Ral, 1), d, **bf)
        pre_al = torch.empty(max(Ral, 1), 2 * F, **bf)
        ws = torch.empty(max(int(L.hep_moe_ffn_workspace(ns, Ral, ns)), 256), dtype=torch.uint8, device=self.device)
        if R > 0:
            ck(L.hep_moe_permute(recv.data_ptr(), row_map.data_ptr(), R, 1, d, rows_al.data_ptr(), s),
               "hep_moe_permute(align)")
        # padding rows are never written by the GEMMs; the weight-gradient GEMMs contract
        # over them (dW13 += dA13^T X, dW2 += dY^T H), so X and H padding must be zero
        ck(L.hep_moe_zero_padding(slot_rows.data_ptr(), seg_al.data_ptr(), ns, ns, rows_al.data_ptr(), d, s),
           "hep_moe_zero_padding(rows)")
        ck(L.hep_moe_zero_padding(slot_rows.data_ptr(), seg_al.data_ptr(), ns, ns, h_al.data_ptr(), F, s),
           "hep_moe_zero_padding(h)")
        ck(L.hep_moe_expert_ffn_train(rows_al.data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(), seg_al.data_ptr(), ns,
                                      Ral, d, F, ns, h_al.data_ptr(), y_al.data_ptr(), pre_al.data_ptr(),
                                      ws.data_ptr(), ws.numel(), rk.sched.status.data_ptr(), s),
           "hep_moe_expert_ffn_train")
        if R > 0:
            ck(L.hep_moe_gather_sum(y_al.data_ptr(), row_map.data_ptr(), None, None, R, 1, d, y.data_ptr(), s),
               "hep_moe_gather_sum(unalign)")
        b.update(row_map=row_map, seg_al=seg_al, slot_rows=slot_rows, Ral=Ral, rows_al=rows_al, h_al=h_al,
                 pre_al=pre_al, ffn_ws=ws, R_recv=R)
        return y[:R]

    def backward(self, douts: list[torch.Tensor], stream=None):
        """Gradients of the last training forward.  douts[i] = dL/dout of rank
        self.ranks[i].  Returns, per driven rank, (dx bf16 [T][d], dWg fp32 [E][d]
        summed over all ranks, dW13 fp32 [n_slots][2F][d], dW2 fp32 [n_slots][d][F])
        where slot s of rank r holds the gradient of expert e (slots[e] = s) summed
        over every replica of e in its EDP group — identical on all replicas."""
        if not self.train_mode:
            raise RuntimeError("construct EPMoELayer(train=True) to run the backward pass")
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            if self.exchange == "p2p":
                return self._backward_p2p(douts, st)
            return self._backward(douts, st)

    def _backward(self, douts, st):
        L = _lib.lib()
        s = st.cuda_stream
        ck = _lib.check
        K, E, G, d, F = self.K, self.E, self.G, self.d, self.F
        dev = self.device
        bs = [rk.buffers(self, b_x.shape[0]) for rk, b_x in zip(self.ranks, douts)]
        dys, dws = [], []
        for rk, b, dout in zip(self.ranks, bs, douts):
            T = dout.shape[0]
            dy = torch.empty(max(T * K, 1), d, dtype=torch.bfloat16, device=dev)
            dw = torch.empty(T, K, dtype=torch.float32, device=dev)
            ck(L.hep_moe_combine_bwd(dout.contiguous().data_ptr(), b["back"].data_ptr(), b["tok_row"].data_ptr(),
                                     b["topk_w"].data_ptr(), T, K, d, dy.data_ptr(), dw.data_ptr(), s),
               "hep_moe_combine_bwd")
            dys.append(dy[: sum(b["send_counts"])])
            dws.append(dw)
        send_counts = [b["send_counts"] for b in bs]
        recv_counts = [b["recv_counts"] for b in bs]
        dy_recvs = self.comm.all_to_all(dys, send_counts, recv_counts)
        dx_recvs, dw13s, dw2s = [], [], []
        for rk, b, dyr in zip(self.ranks, bs, dy_recvs):
            ns, R, Ral = rk.n_slots, b["R_recv"], b["Ral"]
            bf = dict(dtype=torch.bfloat16, device=dev)
            dy_al = torch.empty(max(Ral, 1), d, **bf)
            if R > 0:
                ck(L.hep_moe_permute(dyr.data_ptr(), b["row_map"].data_ptr(), R, 1, d, dy_al.data_ptr(), s),
                   "hep_moe_permute(align)")
            da13 = torch.empty(max(Ral, 1), 2 * F, **bf)
            dx_al = torch.empty(max(Ral, 1), d, **bf)
            dw13 = torch.empty(ns, 2 * F, d, dtype=torch.float32, device=dev)
            dw2 = torch.empty(ns, d, F, dtype=torch.float32, device=dev)
            ck(L.hep_moe_expert_ffn_bwd(b["rows_al"].data_ptr(), b["pre_al"].data_ptr(), b["h_al"].data_ptr(),
                                        dy_al.data_ptr(), rk.w13.data_ptr(), rk.w2.data_ptr(), b["seg_al"].data_ptr(),
                                        ns, b["slot_rows"].data_ptr(), Ral, d, F, ns, da13.data_ptr(),
                                        dx_al.data_ptr(), dw13.data_ptr(), dw2.data_ptr(), b["ffn_ws"].data_ptr(),
                                        b["ffn_ws"].numel(), rk.sched.status.data_ptr(), s),
               "hep_moe_expert_ffn_bwd")
            dxr = torch.empty(max(R, 1), d, **bf)
            if R > 0:
                ck(L.hep_moe_gather_sum(dx_al.data_ptr(), b["row_map"].data_ptr(), None, None, R, 1, d,
                                        dxr.data_ptr(), s), "hep_moe_gather_sum(unalign)")
            dx_recvs.append(dxr[:R])
            dw13s.append(dw13)
            dw2s.append(dw2)
        dx_sends = self.comm.all_to_all(dx_recvs, recv_counts, send_counts)
        dxs, dwgs = [], []
        for b, dxs_rows, dw in zip(bs, dx_sends, dws):
            x = b["x"]
            T = x.shape[0]
            dlogits = torch.empty(T, self.e64, dtype=torch.bfloat16, device=dev)
            dwg = torch.empty(self.e64, d, dtype=torch.float32, device=dev)
            dxg = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            dx = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            ck(L.hep_gate_bwd(b["topk_idx"].data_ptr(), b["topk_w"].data_ptr(), dw.data_ptr(), T, K, self.e64,
                              dlogits.data_ptr(), s), "hep_gate_bwd")
            ck(L.hep_router_bwd(x.data_ptr(), self.wg.data_ptr(), dlogits.data_ptr(), T, d, self.e64,
                                dwg.data_ptr(), dxg.data_ptr(), s), "hep_router_bwd")
            ck(L.hep_moe_gather_sum(dxs_rows.data_ptr(), b["tok_row"].data_ptr(), None, dxg.data_ptr(), T, K, d,
                                    dx.data_ptr(), s), "hep_moe_gather_sum")
            dxs.append(dx)
            dwgs.append(dwg)
        self.comm.all_reduce(dwgs)
        edp_reduce(self.placement, self.comm, [rk.rank for rk in self.ranks], dw13s, dw2s)
        return [(dx, dwg[:E], dw13, dw2) for dx, dwg, dw13, dw2 in zip(dxs, dwgs, dw13s, dw2s)]


def edp_reduce(placement: Placement, comm, ranks: list[int], dw13s: list[torch.Tensor],
               dw2s: list[torch.Tensor]) -> None:
    """Sum every expert's weight gradient over its EDP group (the GPUs holding a
    replica of it), in place, so every replica applies the same update
    (SURVEY.md §8e).  dw13s[i] / dw2s[i] are rank ranks[i]'s
    per-slot gradients [n_slots][2F][d] / [n_slots][d][F] (slot = placement.slots[e]).

    One all-to-all-v carries, from rank r to rank q, the gradients of the experts
    both host (ascending expert id) — no per-group communicators; each replica
    then adds its group's contributions in ascending rank order, so all replicas
    end bit-identical."""
    pl, G = placement, placement.num_gpus
    hosted = [set(h) for h in pl.hosted]
    shp13, shp2 = tuple(dw13s[0].shape[1:]), tuple(dw2s[0].shape[1:])
    n13, n2 = dw13s[0][0].numel(), dw2s[0][0].numel()
    per = n13 + n2
    shared = [[sorted(hosted[r] & hosted[q]) if q != r else [] for q in range(G)] for r in range(G)]
    sends, send_counts, recv_counts = [], [], []
    for r, dw13, dw2 in zip(ranks, dw13s, dw2s):
        parts = []
        for q in range(G):
            for e in shared[r][q]:
                sl = pl.slots[e]
                parts += [dw13[sl].reshape(-1), dw2[sl].reshape(-1)]
        sends.append(torch.cat(parts) if parts else dw13.new_empty(0))
        send_counts.append([len(shared[r][q]) * per for q in range(G)])
        recv_counts.append([len(shared[q][r]) * per for q in range(G)])
    recvs = comm.all_to_all(sends, send_counts, recv_counts)
    for r, dw13, dw2, recv, rc in zip(ranks, dw13s, dw2s, recvs, recv_counts):
        off = _offsets(rc)
        for e in sorted(hosted[r]):
            members = sorted(set(pl.edp_groups[e]))
            if len(members) < 2:
                continue
            sl = pl.slots[e]
            t13 = t2 = None
            for q in members:
                if q == r:
                    g13, g2 = dw13[sl], dw2[sl]
                else:
                    base = off[q] + shared[q][r].index(e) * per
                    g13 = recv[base: base + n13].view(shp13)
                    g2 = recv[base + n13: base + per].view(shp2)
                t13 = g13.clone() if t13 is None else t13.add_(g13)
                t2 = g2.clone() if t2 is None else t2.add_(g2)
            dw13[sl].copy_(t13)
            dw2[sl].copy_(t2)


def migrate_weights(old: Placement, new: Placement, comm, ranks: list[int], old_w13s, old_w2s, new_w13s,
                    new_w2s) -> dict:
    """Move expert weight slots from ``old`` to ``new`` placement.  ``old_*[i]`` /
    ``new_*[i]`` are rank ``ranks[i]``'s slot tensors ([n_slots][...], slot =
    placement.slots[e]).  A replica (e, g) new to the placement is sent by
    src(e) = the lowest GPU in e's old EDP group; all ranks derive the same plan
    from the two placements, so only weights travel (one all-to-all-v)."""
    G = old.num_gpus
    old_sets = [set(g) for g in old.edp_groups]
    src = {}
    moves = [[[] for _ in range(G)] for _ in range(G)]  # moves[q][r]: experts q sends to r (ascending)
    for e, grp in enumerate(new.edp_groups):
        for r in sorted(set(grp)):
            if r in old_sets[e]:
                continue
            if not old_sets[e]:
                raise PlacementError(f"expert {e} has no replica in the old placement to copy from")
            src[e] = min(old_sets[e])
            moves[src[e]][r].append(e)
    for q in range(G):
        for r in range(G):
            moves[q][r].sort()
    sh13, sh2 = tuple(old_w13s[0].shape[1:]), tuple(old_w2s[0].shape[1:])
    n13, n2 = old_w13s[0][0].numel(), old_w2s[0][0].numel()
    per = n13 + n2
    sends, send_counts, recv_counts = [], [], []
    for r, w13, w2, nw13, nw2 in zip(ranks, old_w13s, old_w2s, new_w13s, new_w2s):
        for e in new.hosted[r]:  # replicas staying on this GPU: local slot copy
            if r in old_sets[e]:
                nw13[new.slots[e]].copy_(w13[old.slots[e]])
                nw2[new.slots[e]].copy_(w2[old.slots[e]])
        parts = []
        for q in range(G):
            for e in moves[r][q]:
                parts += [w13[old.slots[e]].reshape(-1), w2[old.slots[e]].reshape(-1)]
        sends.append(torch.cat(parts) if parts else w13.new_empty(0))
        send_counts.append([len(moves[r][q]) * per for q in range(G)])
        recv_counts.append([len(moves[q][r]) * per for q in range(G)])
    recvs = comm.all_to_all(sends, send_counts, recv_counts)
    for r, nw13, nw2, recv, rc in zip(ranks, new_w13s, new_w2s, recvs, recv_counts):
        off = _offsets(rc)
        for q in range(G):
            for j, e in enumerate(moves[q][r]):
                base = off[q] + j * per
                nw13[new.slots[e]].copy_(recv[base: base + n13].view(sh13))
                nw2[new.slots[e]].copy_(recv[base + n13: base + per].view(sh2))
    moved = sum(len(moves[q][r]) for q in range(G) for r in range(G))
    elem = old_w13s[0].element_size()
    return {"moved_replicas": moved, "bytes_sent": sum(sum(c) for c in send_counts) * elem,
            "bytes_per_replica": per * elem}
