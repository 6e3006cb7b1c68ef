"""CPU restatement of the MoE-layer data path (numpy, fp32).

TEST INFRASTRUCTURE ONLY (see oracle/hep_oracle.c header): imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs, never by the package.

The reference models the token data path only as a cost (simulator.py:439-476)
and never models the gate, so the semantics here are the
builder's (documented in paper_2511_16947_b200/layer.py); the schedule they
consume is anchored to the reference through the Dinic oracle
(oracle/hep_oracle.c), and the token -> row rule restates the RoutingTable
contract "for a fixed (expert, src) the ranges appear in routing order and
partition that source's tokens in sequence order" (router.py:38-46).
"""

from __future__ import annotations

import numpy as np

from . import oracle as O


def topk_select(logits: np.ndarray, K: int, bias: np.ndarray | None = None):
    """Top-K of (logit + bias) per row, ties -> lower expert id; weights =
    softmax over the K selected logits (fp32)."""
    T, E = logits.shape
    scores = logits if bias is None else logits + bias[None, :].astype(np.float32)
    # stable argsort on -score keeps lower index first among equal scores
    order = np.argsort(-scores, axis=1, kind="stable")[:, :K].astype(np.int32)
    sel = np.take_along_axis(logits, order, axis=1).astype(np.float32)
    mx = sel.max(axis=1, keepdims=True)
    ex = np.exp((sel - mx).astype(np.float64))
    w = (ex / ex.sum(axis=1, keepdims=True)).astype(np.float32)
    return order, w


def histogram(topk_idx: np.ndarray, E: int, n_src: int, tps: int) -> np.ndarray:
    """hist[src][e] = number of tokens of source src routed to expert e."""
    T = topk_idx.shape[0]
    src = np.minimum(np.arange(T) // tps, n_src - 1)
    h = np.zeros((n_src, E), dtype=np.int64)
    np.add.at(h, (np.repeat(src, topk_idx.shape[1]), topk_idx.reshape(-1)), 1)
    return h


def receive_rows(groups, G: int, xi, ranges, topk_idx: np.ndarray, tps: int):
    """Rows in the [expert asc][dst asc][src asc][rank] receive layout for
    every (token, k); ranks within (src, expert) follow token order."""
    T, K = topk_idx.shape
    E = len(groups)
    base = {}
    row = 0
    expert_rows = np.zeros(E + 1, dtype=np.int64)
    for e in range(E):
        expert_rows[e] = row
        for dst in sorted(groups[e]):
            base[(e, dst)] = row
            row += xi[e][list(groups[e]).index(dst)]
    expert_rows[E] = row
    # per (e, src): list of (rank_end, row_minus_rank) in table order
    lists = {}
    by_e = {}
    for (e, s, d, c) in ranges:
        by_e.setdefault(e, []).append((s, d, c))
    for e, rs in by_e.items():
        for j, (s, d, c) in enumerate(rs):
            r = base[(e, d)] + sum(c2 for (s2, d2, c2) in rs if d2 == d and s2 < s)
            rank = sum(c2 for (s2, d2, c2) in rs[:j] if s2 == s)
            lists.setdefault((e, s), []).append((rank + c, r - rank))
    tok_row = np.zeros((T, K), dtype=np.int64)
    ctr = {}
    for t in range(T):
        s = min(t // tps, G - 1)
        for k in range(K):
            e = int(topk_idx[t, k])
            q = ctr.get((e, s), 0)
            ctr[(e, s)] = q + 1
            lst = lists[(e, s)]
            j = 0
            while j + 1 < len(lst) and q >= lst[j][0]:
                j += 1
            tok_row[t, k] = q + lst[j][1]
    return tok_row, expert_rows


def receive_rows_pipelined(groups, G: int, former, latter, former_loads, topk_idx: np.ndarray, tps: int):
    """Pipelined split (simulator.py:420-435) receive layout [expert][phase][dst][src][rank]:
    expert e's block starts at the prefix of the experts' total loads and holds the static
    phase's rows first; within (expert, src) the first former_loads[e][src] assignments in
    token order belong to the static phase (its ranges), the rest to the scheduled phase
    (its ranges, ranks continuing).  ``former`` / ``latter`` = dict(xi=..., ranges=...)."""
    T, K = topk_idx.shape
    E = len(groups)
    tot = [sum(former["xi"][e]) + sum(latter["xi"][e]) for e in range(E)]
    start = np.concatenate([[0], np.cumsum(tot)]).astype(np.int64)
    lists = {}
    for ph, plan in enumerate((former, latter)):
        base = {}
        for e in range(E):
            row = int(start[e]) + (sum(former["xi"][e]) if ph else 0)
            for dst in sorted(groups[e]):
                base[(e, dst)] = row
                row += plan["xi"][e][list(groups[e]).index(dst)]
        by_e = {}
        for (e, s, d, c) in plan["ranges"]:
            by_e.setdefault(e, []).append((s, d, c))
        for e, rs in by_e.items():
            for j, (s, d, c) in enumerate(rs):
                r = base[(e, d)] + sum(c2 for (s2, d2, c2) in rs if d2 == d and s2 < s)
                rank = (former_loads[e][s] if ph else 0) + sum(c2 for (s2, d2, c2) in rs[:j] if s2 == s)
                lists.setdefault((e, s), []).append((rank, rank + c, r - rank))
    tok_row = np.zeros((T, K), dtype=np.int64)
    ctr = {}
    for t in range(T):
        s = min(t // tps, G - 1)
        for k in range(K):
            e = int(topk_idx[t, k])
            q = ctr.get((e, s), 0)
            ctr[(e, s)] = q + 1
            (hit,) = [lst for lst in lists[(e, s)] if lst[0] <= q < lst[1]]
            tok_row[t, k] = q + hit[2]
    return tok_row, int(start[-1])


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round to nearest even) -> fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def silu(x):
    return x / (1.0 + np.exp(-x))


def expert_ffn(x_rows: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """SwiGLU FFN in fp32 with the bf16 intermediate the device keeps."""
    h = silu(x_rows @ w1.T) * (x_rows @ w3.T)
    return bf16_round(h) @ w2.T


def layer_forward(x, logits, K, groups, G, w1, w2, w3, bias=None, sample=None):
    """Full layer on CPU.  x [T][d] fp32 (bf16 values), logits [T][E] fp32 as
    computed on the device (the oracle's routing decisions are taken on the
    same logits so they are comparable bit for bit).  Returns a dict with every
    intermediate.  ``sample`` restricts the FFN/combine to a subset of tokens."""
    T, E = logits.shape
    tps = T // G
    topk_idx, topk_w = topk_select(logits, K, bias)
    hist = histogram(topk_idx, E, G, tps)
    sched = O.full_path(G, groups, hist.T.copy())
    tok_row, expert_rows = receive_rows(groups, G, sched["xi"], sched["ranges"], topk_idx, tps)
    toks = np.arange(T) if sample is None else np.asarray(sample)
    out = np.zeros((len(toks), x.shape[1]), dtype=np.float32)
    for k in range(K):
        e_of = topk_idx[toks, k]
        for e in np.unique(e_of):
            sel = np.nonzero(e_of == e)[0]
            y = expert_ffn(x[toks[sel]], w1[e], w3[e], w2[e])
            out[sel] += topk_w[toks[sel], k][:, None] * bf16_round(y)
    return dict(topk_idx=topk_idx, topk_w=topk_w, hist=hist, sched=sched, tok_row=tok_row, expert_rows=expert_rows,
                out=out, tokens=toks)
