"""The token-scheduling MoE layer on one B200 (device-resident hot path).

Per micro-batch, all on one CUDA stream, no host synchronisation:

  K1  router GEMM   logits[T][E] = x . Wg^T, with the    hep_router_topk (tcgen05; gate in the
      + gate        top-K + softmax(top-K) + hist[G][E]  epilogue, one TMEM lane per token)
  K3  scheduler     m, lex-min plan, integerize, ranges hep_sched_solve (1 CTA)
  K4  assignment    (token, k) -> receive row           hep_moe_assign_precounted
  K5  permute       rows[row] = x[token]                hep_moe_permute (128-bit, one warp per token)
  K6  expert FFN    SwiGLU grouped GEMM x2              hep_moe_expert_ffn (tcgen05; opt-in
                                                        hep_moe_expert_ffn_gather fuses K5)
  K7  combine       out[t] = sum_k w * y[row]           hep_moe_combine

``MoELayer`` with ``num_sources = G`` runs the paper's EP group of G GPUs
*simulated on one device* (the reference's own "simulated EP" setting,
BASELINE configs[0]): tokens [g*T/G, (g+1)*T/G) originate on virtual GPU g,
the scheduler balances the G virtual GPUs exactly as on G real ones, the
dispatch "all-to-all" is the K5 scatter into the [expert][dst][src] receive
layout, and every virtual GPU's replicas run in one grouped GEMM (one
physical weight copy per expert; replicas of an expert are identical by
construction).  The schedule — routing decisions, per-GPU
loads, token-to-GPU assignment — is the same bit-exact object the
multi-GPU layer uses.

Semantics owned by this builder (the reference never models the gate,
SPEC.md:499): selection = top-K of (logit + bias_e) with ties to the lower
expert id; weights = softmax over the K selected logits; expert =
SwiGLU FFN  y = (silu(x W1^T) * (x W3^T)) W2^T  with a bf16 intermediate.
"""

from __future__ import annotations

import ctypes
from fractions import Fraction

import torch

from . import _lib
from .core import Placement
from .scheduler import HEP_SCHED_ALL, DeviceScheduler


def interleave_w13(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[E][F][d] x2 -> [E][2F][d] with 128-row blocks alternating W1, W3 (the
    layout the fused SwiGLU epilogue expects, include/hep.h)."""
    E, F, d = w1.shape
    assert F % 128 == 0
    a = w1.reshape(E, F // 128, 128, d)
    b = w3.reshape(E, F // 128, 128, d)
    return torch.stack((a, b), dim=2).reshape(E, 2 * F, d).contiguous()


def init_expert_weights(num_experts: int, d_model: int, ffn: int, seed: int, device, dtype=torch.bfloat16):
    """W1, W3 ~ N(0, 1/d), W2 ~ N(0, 1/F), seeded by expert id
    so every replica of an expert is identical."""
    w1 = torch.empty(num_experts, ffn, d_model, dtype=dtype, device=device)
    w3 = torch.empty_like(w1)
    w2 = torch.empty(num_experts, d_model, ffn, dtype=dtype, device=device)
    for e in range(num_experts):
        g = torch.Generator(device=device).manual_seed(seed * 100003 + e)
        w1[e].copy_(torch.randn(ffn, d_model, generator=g, device=device) / d_model ** 0.5)
        w3[e].copy_(torch.randn(ffn, d_model, generator=g, device=device) / d_model ** 0.5)
        w2[e].copy_(torch.randn(d_model, ffn, generator=g, device=device) / ffn ** 0.5)
    return w1, w2, w3


class MoEBuffers:
    """All device buffers of one micro-batch shape, allocated once (the hot
    path allocates nothing; CUDA-graph capturable)."""

    def __init__(self, sched: DeviceScheduler, T: int, K: int, E: int, e_pad: int, d_model: int, ffn: int, device,
                 train: bool = False, pipelined: bool = False):
        L = _lib.lib()
        G = sched.G
        # training keeps every expert block 64-row aligned (weight-gradient GEMMs contract
        # over whole 64-row blocks); padding rows are never written, so the row buffers
        # start zeroed (a padding row only ever holds zeros or an older finite row)
        self.row_align = 64 if train else 1
        R = T * K + (E * 63 if train else 0)
        self.R = R
        alloc = torch.zeros if train else torch.empty
        bf = dict(dtype=torch.bfloat16, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        self.logits = torch.empty(T, e_pad, dtype=torch.float32, device=device)
        self.topk_idx = torch.empty(T, K, **i32)
        self.topk_w = torch.empty(T, K, dtype=torch.float32, device=device)
        self.hist = torch.zeros(G, E, dtype=torch.int64, device=device)
        # hep_router_topk_ws: the router kernel zeroes hist itself through these (self-resetting)
        self.router_sync = torch.zeros(4, dtype=torch.int32, device=device)
        self.tok_row = torch.empty(T, K, **i32)
        self.row_tok = torch.empty(max(R, 1), **i32)
        # pipelined split: [expert][phase][dst][src][rank], one segment list per phase; the two
        # phases' assignments run on two streams, each with its own workspace and row map
        self.n_seg = sched.nnz * (2 if pipelined else 1)
        self.seg = torch.empty(max(self.n_seg, 1), 4, **i32)
        self.expert_rows = torch.empty(E + 1, dtype=torch.int64, device=device)
        self.expert_rows2 = torch.empty(E + 1, dtype=torch.int64, device=device) if pipelined else None
        ws = L.hep_moe_assign_workspace(sched.handle, T, K)
        self.assign_ws = torch.empty(max(int(ws), 256), dtype=torch.uint8, device=device)
        self.assign_ws2 = torch.empty(max(int(ws), 256), dtype=torch.uint8, device=device) if pipelined else None
        self.tok_row_ph = [torch.empty(T, K, **i32) for _ in range(2)] if pipelined else None
        self.chunk_off = int(L.hep_moe_assign_chunk_offset(sched.handle, T, K))  # router-written chunk counts
        self.rows = alloc(max(R, 1), d_model, **bf)
        self.h = alloc(max(R, 1), ffn, **bf)
        self.y = alloc(max(R, 1), d_model, **bf)
        fws = L.hep_moe_ffn_workspace(max(self.n_seg, 1), R, E)
        self.ffn_ws = torch.empty(max(int(fws), 256), dtype=torch.uint8, device=device)
        self.out = torch.empty(T, d_model, **bf)
        self.pre = torch.zeros(max(R, 1), 2 * ffn, **bf) if train else None


class MoELayer(torch.nn.Module):
    """HarmonyEP MoE layer over a placement of ``placement.num_gpus`` (virtual)
    GPUs, forward pass entirely in sm_100a kernels."""

    def __init__(self, placement: Placement, d_model: int, ffn: int, top_k: int, *, seed: int = 0,
                 gate_bias: torch.Tensor | None = None, device=None, train: bool = False,
                 pipeline_ratio: float | Fraction | None = None, fuse_permute: bool = False):
        super().__init__()
        self.train_mode = train
        # harmony_pipelined (simulator.py:17-20, :375, :420-435): a 1 - pipeline_ratio
        # static share is split evenly over each expert's replicas and assigned before
        # the scheduled share is solved (gpu_base = the static share's GPU loads)
        self.static_share = None
        if pipeline_ratio is not None:
            if not (0.0 < float(pipeline_ratio) <= 1.0):
                raise ValueError("pipeline_ratio must be in (0, 1]")  # SimulationConfig (simulator.py:117-118)
            if train:
                raise ValueError("the pipelined split is a forward (serving) schedule; train with pipeline_ratio=None")
            self.static_share = Fraction(1) - Fraction(pipeline_ratio)
        # fuse_permute: gather the x rows inside the first expert GEMM (TMA tile::gather4)
        # instead of the K5 permute kernel.  Bit-identical, but measured slower (gather4
        # issues one 128-byte row request at a time, ~10 B/clk/SM: Qwen3 FFN 2.15 -> 4.67 ms,
        # profiles/r01/ffn_ab_r01d.txt), so the permute kernel is the default.  Never in
        # training (the weight gradients contract over the permuted rows).
        self.fuse_permute = fuse_permute and not train
        # pipelined: split + 2 scheduler launches, 2 x 4 assignment kernels, 2 permutes
        self.LAUNCHES_PER_FORWARD = (11 if self.static_share is None else 19) - (
            (1 if self.static_share is None else 2) if self.fuse_permute else 0)
        torch_ = _lib.require_cuda()
        self.device = torch_.device("cuda", torch_.cuda.current_device()) if device is None else torch_.device(device)
        self.placement = placement
        self.G = placement.num_gpus
        self.E = placement.num_experts
        self.K = top_k
        self.d = d_model
        self.F = ffn
        if d_model % 256 or ffn % 128:
            raise ValueError("d_model must be a multiple of 256 and ffn a multiple of 128")
        self.e_pad = max(16, (self.E + 15) // 16 * 16)
        self.sched = DeviceScheduler(placement, device=self.device)
        g = torch.Generator(device=self.device).manual_seed(seed * 7919 + 17)
        self.e64 = (self.E + 63) // 64 * 64  # router rows padded to 64 for its backward GEMMs
        wg = torch.zeros(self.e64, d_model, dtype=torch.bfloat16, device=self.device)
        wg[: self.E] = (torch.randn(self.E, d_model, generator=g, device=self.device) / d_model ** 0.5).to(torch.bfloat16)
        self.wg = wg
        w1, w2, w3 = init_expert_weights(self.E, d_model, ffn, seed, self.device)
        self.w1, self.w3 = w1, w3
        self.w13 = interleave_w13(w1, w3)
        self.w2 = w2
        self.gate_bias = None if gate_bias is None else gate_bias.to(self.device, torch.float32).contiguous()
        self._bufs: dict[int, MoEBuffers] = {}
        if self.static_share is not None:
            # the static phase's assignment + dispatch run on a side stream while the scheduled
            # phase is solved (simulator.py:451-453); events fork and join it
            self._side = torch.cuda.Stream(device=self.device)
            self._ev_join = torch.cuda.Event()
        # pipelined split: resident 256-thread blocks per SM of the static phase's permute (8 =
        # all; fewer leave room for the scheduled phase's solve and assignment, which run
        # concurrently on the main stream)
        self.static_permute_blocks_per_sm = 8  # measured: fewer does not shorten the chain (profiles/r02/pipelined_timeline_r02i.txt)

    def set_placement(self, placement: Placement) -> None:
        """Adopt a new placement (adaptive replacement, ``adaptive.py``).  The
        simulated EP group keeps one weight copy per expert, so only the
        device scheduler tables change; buffers are re-sized lazily."""
        if (placement.num_gpus, placement.num_experts) != (self.G, self.E):
            raise ValueError("placement must keep the number of GPUs and experts")
        self.placement = placement
        self.sched = DeviceScheduler(placement, device=self.device)
        self._bufs.clear()

    @torch.no_grad()
    def schedule(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """K1 + K3 only (router GEMM with the fused gate, then the scheduler) on ``x``:
        the micro-batch's histogram, exact schedule, routing and transfer plan on the
        device without moving tokens (balance studies; the schedule is the one a full
        forward computes).  Returns the device tensor of integerized per-GPU loads [G]."""
        if self.static_share is not None:
            raise ValueError("schedule() covers the single-phase harmony schedule")
        L = _lib.lib()
        st = stream if stream is not None else torch.cuda.current_stream()
        T, K, E, G = x.shape[0], self.K, self.E, self.G
        b = self.buffers(T)
        _lib.check(L.hep_router_topk_ws(x.data_ptr(), self.wg.data_ptr(), T, self.d, E, self.e_pad,
                                        _lib.ptr(self.gate_bias), K, T // G, G, b.logits.data_ptr(),
                                        b.topk_idx.data_ptr(), b.topk_w.data_ptr(), b.hist.data_ptr(), None,
                                        b.router_sync.data_ptr(), st.cuda_stream), "hep_router_topk")
        _lib.check(L.hep_sched_solve(self.sched.handle, b.hist.data_ptr(), 1, E, None, HEP_SCHED_ALL,
                                     ctypes.byref(self.sched.out), st.cuda_stream), "hep_sched_solve")
        return self.sched.gpu_load

    def expert_loads(self, T: int) -> list[int]:
        """Per-expert token counts of the last micro-batch (host copy of the
        device histogram's column sums; for the adaptive policy)."""
        return self.buffers(T).hist.sum(dim=0).cpu().tolist()

    def buffers(self, T: int) -> MoEBuffers:
        b = self._bufs.get(T)
        if b is None:
            b = MoEBuffers(self.sched, T, self.K, self.E, self.e_pad, self.d, self.F, self.device, self.train_mode,
                           self.static_share is not None)
            self._bufs[T] = b
        return b

    @torch.no_grad()
    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """x [T][d] bf16 on the device, T divisible by G (tokens of virtual GPU g
        are rows [g*T/G, (g+1)*T/G)).  Returns a view of the layer's output buffer."""
        T = x.shape[0]
        if x.dtype != torch.bfloat16 or x.shape[1] != self.d or not x.is_contiguous():
            raise ValueError("x must be a contiguous [T, d_model] bf16 tensor")
        if T % self.G:
            raise ValueError(f"T={T} must be divisible by the {self.G} source GPUs")
        b = self.buffers(T)
        self.run(x, b, stream)
        return b.out

    def run(self, x: torch.Tensor, b: MoEBuffers, stream=None, events: dict | None = None,
            dispatch_only: bool = False) -> None:
        """Launch the whole forward chain on `stream`.  ``events`` optionally maps
        a stage name ("router", "gate", "sched", "assign", "permute", "ffn",
        "combine") to a (start, end) pair of torch.cuda.Event recorded around it.
        ``dispatch_only``: stop after the permute (timing of the scheduling chain)."""
        L = _lib.lib()
        st = stream if stream is not None else torch.cuda.current_stream()
        s = st.cuda_stream
        T, K, E, G = x.shape[0], self.K, self.E, self.G
        tps = T // G
        ck = _lib.check
        ev = events or {}

        def mark(name, i):
            pair = ev.get(name)
            if pair is not None:
                pair[i].record(st)

        # K1: router GEMM with the gate (top-K, weights, histogram, per-chunk counts) fused
        # into its epilogue; the logits are also written (parity tests, inspection)
        mark("router", 0)
        chunk = None if self.static_share is not None else b.assign_ws.data_ptr() + b.chunk_off
        ck(L.hep_router_topk_ws(x.data_ptr(), self.wg.data_ptr(), T, self.d, E, self.e_pad, _lib.ptr(self.gate_bias),
                                K, tps, G, b.logits.data_ptr(), b.topk_idx.data_ptr(), b.topk_w.data_ptr(),
                                b.hist.data_ptr(), chunk, b.router_sync.data_ptr(), s), "hep_router_topk")
        mark("router", 1)
        mark("gate", 0)  # fused into the router kernel
        mark("gate", 1)
        # hist is [G][E] (source-major, the all-gather layout): stride_e = 1, stride_g = E
        mark("sched", 0)
        if self.static_share is None:
            ck(L.hep_sched_solve(self.sched.handle, b.hist.data_ptr(), 1, E, None, HEP_SCHED_ALL,
                                 ctypes.byref(self.sched.out), s), "hep_sched_solve")
        else:
            # the static phase's routing runs on the side stream, forked after the split, while
            # the scheduled phase is solved here
            self.sched.launch_pipelined(b.hist, 1, E, self.static_share, HEP_SCHED_ALL, st, stream_static=self._side)
        mark("sched", 1)
        mark("assign", 0)
        if self.static_share is None:
            ck(L.hep_moe_assign_precounted(self.sched.handle, ctypes.byref(self.sched.out), b.topk_idx.data_ptr(), T,
                                           K, tps, b.row_align, b.tok_row.data_ptr(), b.row_tok.data_ptr(),
                                           b.seg.data_ptr(), b.expert_rows.data_ptr(), b.assign_ws.data_ptr(),
                                           b.assign_ws.numel(), s), "hep_moe_assign_precounted")
            mark("assign", 1)
            mark("permute", 0)
            if not self.fuse_permute:
                ck(L.hep_moe_permute(x.data_ptr(), b.tok_row.data_ptr(), T, K, self.d, b.rows.data_ptr(), s),
                   "hep_moe_permute")
            mark("permute", 1)
        else:
            # harmony_pipelined: the static phase's routing, assignment and dispatch (permute)
            # run on the side stream, overlapping the scheduled phase's solve, assignment and
            # permute on this stream (simulator.py:420-435, :451-453).  The two phases write
            # disjoint entries of tok_row / row_tok / seg and disjoint rows.
            nnz = self.sched.nnz
            split = self.sched.split.data_ptr()
            side = self._side
            ss = side.cuda_stream
            tr0 = None if self.fuse_permute else b.tok_row_ph[0].data_ptr()
            ck(L.hep_moe_assign_phase(self.sched.handle, ctypes.byref(self.sched.former.out), split, 0,
                                      b.topk_idx.data_ptr(), T, K, tps, b.tok_row.data_ptr(), tr0,
                                      b.row_tok.data_ptr(), b.seg.data_ptr(), b.expert_rows.data_ptr(),
                                      b.assign_ws2.data_ptr(), b.assign_ws2.numel(), ss),
               "hep_moe_assign_phase(static)")
            if not self.fuse_permute:
                # capped occupancy: SM room for the solve / assignment running on the main stream
                ck(L.hep_moe_permute_ex(x.data_ptr(), tr0, T, K, self.d, b.rows.data_ptr(),
                                        self.static_permute_blocks_per_sm, ss), "hep_moe_permute(static)")
            self._ev_join.record(side)
            tr1 = None if self.fuse_permute else b.tok_row_ph[1].data_ptr()
            ck(L.hep_moe_assign_phase(self.sched.handle, ctypes.byref(self.sched.out), split, 1,
                                      b.topk_idx.data_ptr(), T, K, tps, b.tok_row.data_ptr(), tr1,
                                      b.row_tok.data_ptr(), b.seg.data_ptr() + 16 * nnz, b.expert_rows2.data_ptr(),
                                      b.assign_ws.data_ptr(), b.assign_ws.numel(), s),
               "hep_moe_assign_phase(scheduled)")
            mark("assign", 1)
            mark("permute", 0)
            if not self.fuse_permute:
                ck(L.hep_moe_permute(x.data_ptr(), tr1, T, K, self.d, b.rows.data_ptr(), s), "hep_moe_permute(scheduled)")
            st.wait_event(self._ev_join)  # both phases' rows and segments are in place
            mark("permute", 1)
        if dispatch_only:
            return
        mark("ffn", 0)
        if self.fuse_permute:  # K5 fused into GEMM 1: x rows gathered by TMA through row_tok
            ck(L.hep_moe_expert_ffn_gather(x.data_ptr(), T, b.row_tok.data_ptr(), self.w13.data_ptr(),
                                           self.w2.data_ptr(), b.seg.data_ptr(), b.n_seg, b.R, self.d, self.F, E,
                                           b.h.data_ptr(), b.y.data_ptr(), b.ffn_ws.data_ptr(), b.ffn_ws.numel(),
                                           self.sched.status.data_ptr(), s), "hep_moe_expert_ffn_gather")
        elif b.pre is None:
            ck(L.hep_moe_expert_ffn(b.rows.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(), b.seg.data_ptr(),
                                    b.n_seg, b.R, self.d, self.F, E, b.h.data_ptr(), b.y.data_ptr(),
                                    b.ffn_ws.data_ptr(), b.ffn_ws.numel(), self.sched.status.data_ptr(), s),
               "hep_moe_expert_ffn")
        else:
            ck(L.hep_moe_expert_ffn_train(b.rows.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(),
                                          b.seg.data_ptr(), self.sched.nnz, b.R, self.d, self.F, E, b.h.data_ptr(),
                                          b.y.data_ptr(), b.pre.data_ptr(), b.ffn_ws.data_ptr(), b.ffn_ws.numel(),
                                          self.sched.status.data_ptr(), s), "hep_moe_expert_ffn_train")
        mark("ffn", 1)
        mark("combine", 0)
        ck(L.hep_moe_combine(b.y.data_ptr(), b.tok_row.data_ptr(), b.topk_w.data_ptr(), T, K, self.d,
                             b.out.data_ptr(), s), "hep_moe_combine")
        mark("combine", 1)

    def capture(self, x: torch.Tensor, dispatch_only: bool = False) -> "torch.cuda.CUDAGraph":
        """Record one forward on ``x`` (fixed buffers, no host sync anywhere in the
        chain) as a CUDA graph; ``graph.replay()`` re-runs all 11 kernels with one
        launch.  ``x`` must stay the input tensor (refill it in place).
        ``dispatch_only``: the chain up to the permute only (see ``run``)."""
        b = self.buffers(x.shape[0])
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm the launch paths (attributes, tensor maps) outside the capture
            self.run(x, b, side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self.run(x, b, side, dispatch_only=dispatch_only)
        return g

    # kernels launched per forward: router GEMM + gate epilogue, scheduler, assign x3
    # (plan prep, chunk scan, chunk map; the chunk counts come from the router epilogue),
    # permute, FFN (tile count + tile list + 2 GEMMs), combine (pipelined split: + split
    # kernel, second scheduler launch, per-phase assignment x4 each)
    LAUNCHES_PER_FORWARD = 11

    def launches_per_forward(self, T: int) -> int:
        """Kernels one forward on T tokens launches (LAUNCHES_PER_FORWARD counts the FFN as
        4; with many light experts it runs them as a second 1-CTA GEMM pair: 8)."""
        L = _lib.lib()
        return self.LAUNCHES_PER_FORWARD - 4 + int(L.hep_moe_ffn_launches(T * self.K, self.E, int(self.fuse_permute)))

    def check_status(self):
        self.sched.check_status("MoELayer")

    # ------------------------------------------------------------------ training
    def backward_step(self, x: torch.Tensor, dout: torch.Tensor, stream=None):
        """Gradients of the last forward on ``x`` (training mode), all on the device:
        returns (dx bf16 [T][d], dWg fp32 [E][d], dW13 fp32 [E][2F][d] (W13
        interleave), dW2 fp32 [E][d][F]).

          K7^T  dY rows = w * dout, dw = <dout, Y>                hep_moe_combine_bwd
          K6^T  dA13 = swiglu'(A13) * (dY W2), dX rows = dA13 W13,
                dW2 = dY^T H, dW13 = dA13^T X  (per expert)       hep_moe_expert_ffn_bwd
          K1^T  dlogits = w (dw - sum w dw) on the selected experts,
                dWg = dlogits^T x, dx_gate = dlogits Wg           hep_gate_bwd, hep_router_bwd
          K5^T  dx = dx_gate + sum_k dX[row(t,k)]                 hep_moe_gather_sum
        """
        if not self.train_mode:
            raise RuntimeError("construct MoELayer(train=True) to run the backward pass")
        L = _lib.lib()
        st = stream if stream is not None else torch.cuda.current_stream()
        s = st.cuda_stream
        ck = _lib.check
        T, K, E, d, F = x.shape[0], self.K, self.E, self.d, self.F
        b = self.buffers(T)
        dout = dout.contiguous()
        dev = self.device
        with torch.cuda.stream(st):
            dy = torch.empty_like(b.y)
            dw = torch.empty(T, K, dtype=torch.float32, device=dev)
            da13 = torch.empty_like(b.pre)
            dx_rows = torch.empty_like(b.rows)
            dw13 = torch.empty(E, 2 * F, d, dtype=torch.float32, device=dev)
            dw2 = torch.empty(E, d, F, dtype=torch.float32, device=dev)
            dlogits = torch.empty(T, self.e64, dtype=torch.bfloat16, device=dev)
            dwg = torch.empty(self.e64, d, dtype=torch.float32, device=dev)
            dxg = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            dx = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        ck(L.hep_moe_combine_bwd(dout.data_ptr(), b.y.data_ptr(), b.tok_row.data_ptr(), b.topk_w.data_ptr(), T, K, d,
                                 dy.data_ptr(), dw.data_ptr(), s), "hep_moe_combine_bwd")
        ck(L.hep_moe_expert_ffn_bwd(b.rows.data_ptr(), b.pre.data_ptr(), b.h.data_ptr(), dy.data_ptr(),
                                    self.w13.data_ptr(), self.w2.data_ptr(), b.seg.data_ptr(), self.sched.nnz,
                                    b.expert_rows.data_ptr(), b.R, d, F, E, da13.data_ptr(), dx_rows.data_ptr(),
                                    dw13.data_ptr(), dw2.data_ptr(), b.ffn_ws.data_ptr(), b.ffn_ws.numel(),
                                    self.sched.status.data_ptr(), s), "hep_moe_expert_ffn_bwd")
        ck(L.hep_gate_bwd(b.topk_idx.data_ptr(), b.topk_w.data_ptr(), dw.data_ptr(), T, K, self.e64,
                          dlogits.data_ptr(), s), "hep_gate_bwd")
        ck(L.hep_router_bwd(x.data_ptr(), self.wg.data_ptr(), dlogits.data_ptr(), T, d, self.e64, dwg.data_ptr(),
                            dxg.data_ptr(), s), "hep_router_bwd")
        ck(L.hep_moe_gather_sum(dx_rows.data_ptr(), b.tok_row.data_ptr(), None, dxg.data_ptr(), T, K, d,
                                dx.data_ptr(), s), "hep_moe_gather_sum")
        return dx, dwg[:E], dw13, dw2

    def launches_per_backward(self, T: int) -> int:
        """Kernels one backward_step on T tokens launches: combine^T, the expert-FFN backward
        (hep_moe_ffn_bwd_launches: zero padding x2, tile lists, 4 GEMMs, weight-gradient
        expert order, + the light-expert split), gate^T, the router backward (2 GEMMs, + the
        split-K sum when its contraction is split) and the gather-sum."""
        L = _lib.lib()
        R = self.buffers(T).R
        e64, d = self.e64, self.d
        tiles = (e64 + 127) // 128 * (d // 256)
        S = min(L.hep_device_sm_count() // max(tiles, 1), T // (2 * e64), T // 64)
        router = 2 + (1 if S > 1 else 0)
        return 1 + int(L.hep_moe_ffn_bwd_launches(R, self.E)) + 1 + router + 1


class MoEFunction(torch.autograd.Function):
    """Autograd wrapper: forward and backward entirely in the layer's kernels.
    Gradients flow to x and to the layer's parameters (wg, w13, w2)."""

    @staticmethod
    def forward(ctx, x, wg, w13, w2, layer):
        out = layer(x).clone()
        ctx.layer = layer
        ctx.save_for_backward(x)
        return out

    @staticmethod
    def backward(ctx, dout):
        (x,) = ctx.saved_tensors
        layer = ctx.layer
        dx, dwg, dw13, dw2 = layer.backward_step(x, dout.to(torch.bfloat16))
        gwg = torch.zeros_like(layer.wg)
        gwg[: layer.E] = dwg.to(gwg.dtype)
        return dx, gwg, dw13.to(layer.w13.dtype), dw2.to(layer.w2.dtype), None


class HostPipeline:
    """Serving-style public entry point for host-resident micro-batches.

    ``submit(x_host)`` copies a pinned host batch to the device on a copy
    stream, runs the layer on the compute stream and copies the output back
    into a pinned host buffer on a third stream; two device buffer sets are
    rotated so the H2D copy of batch i+1 and the D2H copy of batch i-1
    overlap the layer's kernels of batch i.  ``result(i)`` blocks until
    batch i's output is in host memory.
    """

    def __init__(self, layer: MoELayer, T: int, depth: int = 2):
        self.layer = layer
        dev = layer.device
        self.T = T
        self.depth = depth
        self.x_dev = [torch.empty(T, layer.d, dtype=torch.bfloat16, device=dev) for _ in range(depth)]
        self.bufs = [MoEBuffers(layer.sched, T, layer.K, layer.E, layer.e_pad, layer.d, layer.F, dev,
                                pipelined=layer.static_share is not None) for _ in range(depth)]
        self.out_host = [torch.empty(T, layer.d, dtype=torch.bfloat16).pin_memory() for _ in range(depth)]
        self.s_in = torch.cuda.Stream(device=dev)
        self.s_comp = torch.cuda.Stream(device=dev)
        self.s_out = torch.cuda.Stream(device=dev)
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.n = 0

    def submit(self, x_host: torch.Tensor) -> int:
        i = self.n % self.depth
        if self.n >= self.depth:  # slot reuse: the previous occupant must be fully drained
            self.s_in.wait_event(self.ev_comp[i])
            self.s_comp.wait_event(self.ev_out[i])
        with torch.cuda.stream(self.s_in):
            self.x_dev[i].copy_(x_host, non_blocking=True)
            self.ev_in[i].record(self.s_in)
        self.s_comp.wait_event(self.ev_in[i])
        self.layer.run(self.x_dev[i], self.bufs[i], self.s_comp)
        self.ev_comp[i].record(self.s_comp)
        self.s_out.wait_event(self.ev_comp[i])
        with torch.cuda.stream(self.s_out):
            self.out_host[i].copy_(self.bufs[i].out, non_blocking=True)
            self.ev_out[i].record(self.s_out)
        self.n += 1
        return self.n - 1

    def result(self, ticket: int, copy: bool = False) -> torch.Tensor:
        """Batch ``ticket``'s output in host memory.  Without ``copy`` this is the pinned
        slot buffer itself: valid until ``depth`` more batches are submitted (the slot's
        next D2H copy overwrites it); ``copy=True`` returns a private clone.  Raises for a
        ticket whose slot was already reused."""
        if ticket < 0 or ticket >= self.n:
            raise ValueError(f"ticket {ticket} was never submitted")
        if ticket < self.n - self.depth:
            raise RuntimeError(f"ticket {ticket}: its slot was reused by ticket {ticket + self.depth} "
                               f"(results live for {self.depth} submits; use result(..., copy=True) earlier)")
        i = ticket % self.depth
        self.ev_out[i].synchronize()
        return self.out_host[i].clone() if copy else self.out_host[i]

    def drain(self):
        for e in self.ev_out:
            e.synchronize()
