"""Tensor parallelism for the decode step (Llama-2-70B
at t = 2/4/8 B200s).

Megatron-style sharding of one decoder layer over t ranks:

* QKV: column-parallel by KV-head groups.  Rank r owns query heads
  [r Hq/t, (r+1) Hq/t) and KV heads [r Hkv/t, (r+1) Hkv/t); with GQA the
  query heads of a KV head stay on its rank (G = Hq/Hkv per KV head
  throughout), so attention is local and split-KV never crosses GPUs.  The
  local weight keeps the fused layout [q heads | k heads | v heads] that the
  QKV epilogue (RoPE + KV append, one 128-row tile per head) expects.
* gate|up: column-parallel, local [gate_r | up_r] (the SiLU*up kernel reads
  [gate | up] per token).
* O and down: row-parallel (their K dimension is sharded); each produces a
  partial residual-stream update, summed by ONE all-reduce of [B, hidden]
  per projection.  Rank 0 adds the residual in its epilogue, the others write
  their bare partial in place, so the all-reduce yields x + sum_r partial_r.
* Embedding, final RMSNorm and the LM head are replicated (the argmax is then
  identical on every rank).

The reference has no multi-GPU path; this module is the B200
design for config 5.  ``reference_step`` restates one decode step in torch
fp32 so the sharding (and the all-reduce placement) can be checked on CPU
with a gloo process group against the unsharded model (tests/test_tp.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class ShardDims:
    tp: int
    n_heads: int      # local query heads
    n_kv_heads: int   # local KV heads
    ffn: int          # local FFN width


def shard_dims(cfg, tp: int) -> ShardDims:
    if tp < 1:
        raise ValueError(f"tensor-parallel size must be >= 1, got {tp}")
    if cfg.n_kv_heads % tp or cfg.n_heads % tp or cfg.ffn % tp:
        raise ValueError(f"{cfg.name}: heads ({cfg.n_heads}/{cfg.n_kv_heads}) and ffn ({cfg.ffn}) "
                         f"must divide by tp={tp}")
    f = cfg.ffn // tp
    if f % 8:
        raise ValueError(f"local ffn {f} must be a multiple of 8 (GEMM K alignment)")
    return ShardDims(tp, cfg.n_heads // tp, cfg.n_kv_heads // tp, f)


def rank_gemm_shapes(cfg, tp: int):
    """[N, K] of each dispatched GEMM on one rank."""
    s = shard_dims(cfg, tp)
    D = cfg.head_dim
    return {"qkv": ((s.n_heads + 2 * s.n_kv_heads) * D, cfg.hidden), "o": (cfg.hidden, s.n_heads * D),
            "gate_up": (2 * s.ffn, cfg.hidden), "down": (cfg.hidden, s.ffn),
            "lm_head": (cfg.vocab, cfg.hidden)}


def _rows(w, lo, hi):
    return w[lo:hi]


def shard_qkv(w, cfg, rank: int, tp: int):
    """w: [(Hq + 2 Hkv) D, hidden] (q heads, then k heads, then v heads)."""
    import torch
    s = shard_dims(cfg, tp)
    D, Hq, Hkv = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    q = _rows(w, rank * s.n_heads * D, (rank + 1) * s.n_heads * D)
    k0 = Hq * D
    k = _rows(w, k0 + rank * s.n_kv_heads * D, k0 + (rank + 1) * s.n_kv_heads * D)
    v0 = (Hq + Hkv) * D
    v = _rows(w, v0 + rank * s.n_kv_heads * D, v0 + (rank + 1) * s.n_kv_heads * D)
    return torch.cat([q, k, v], 0).contiguous()


def shard_gate_up(w, cfg, rank: int, tp: int):
    """w: [2 ffn, hidden] = [gate; up]."""
    import torch
    f = shard_dims(cfg, tp).ffn
    return torch.cat([w[rank * f:(rank + 1) * f], w[cfg.ffn + rank * f:cfg.ffn + (rank + 1) * f]], 0).contiguous()


def shard_o(w, cfg, rank: int, tp: int):
    """w: [hidden, Hq D]: the K columns of this rank's query heads."""
    c = shard_dims(cfg, tp).n_heads * cfg.head_dim
    return w[:, rank * c:(rank + 1) * c].contiguous()


def shard_down(w, cfg, rank: int, tp: int):
    """w: [hidden, ffn]: the K columns of this rank's FFN slice."""
    f = shard_dims(cfg, tp).ffn
    return w[:, rank * f:(rank + 1) * f].contiguous()


def shard_layer(layer: dict, cfg, rank: int, tp: int) -> dict:
    """Full layer weights ([N, K] row-major tensors) -> this rank's shard."""
    return {"qkv": shard_qkv(layer["qkv"], cfg, rank, tp), "o": shard_o(layer["o"], cfg, rank, tp),
            "gate_up": shard_gate_up(layer["gate_up"], cfg, rank, tp),
            "down": shard_down(layer["down"], cfg, rank, tp),
            "ln1": layer["ln1"], "ln2": layer["ln2"]}


def shard_cache(cache, cfg, rank: int, tp: int):
    """[B, Hkv, L, D] -> this rank's KV heads."""
    h = shard_dims(cfg, tp).n_kv_heads
    return cache[:, rank * h:(rank + 1) * h].contiguous()


# ----------------------------------------------------------------- fp32 reference
def _rmsnorm(x, w, eps):
    import torch
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _rope(x, pos, theta):
    """x [B, H, D], rotate-half RoPE at positions pos [B] (the QKV epilogue's form)."""
    import torch
    D = x.shape[-1]
    half = D // 2
    inv = theta ** (-2.0 * torch.arange(half, dtype=torch.float64, device=x.device) / D)
    ang = pos.to(x.device).double()[:, None] * inv[None, :]
    cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    x0, x1 = x[..., :half], x[..., half:]
    return torch.cat([x0 * cos - x1 * sin, x1 * cos + x0 * sin], -1)


def reference_layer(x, L: dict, kc, vc, pos, lens, cfg, n_heads, n_kv_heads, *, rank=0, all_reduce=None,
                    trace=None):
    """One decode layer in fp32 on (possibly sharded) weights, on x's device.

    x [B, hidden]; L: qkv [Nq, hidden], o [hidden, Hq_l D], gate_up, down, ln1,
    ln2; kc/vc [B, Hkv_l, Lmax, D] (row pos[b] is written); lens [B] attended
    lengths (pos + 1).  With all_reduce (tp > 1) the O / down outputs are
    partials: rank 0 adds the residual, then all_reduce sums them in place.
    trace: optional dict receiving the intermediates q, k, v (after RoPE) and
    att (the attention output)."""
    import torch
    B = x.shape[0]
    D = cfg.head_dim
    h = _rmsnorm(x, L["ln1"].float(), cfg.eps)
    qkv = h @ L["qkv"].float().T
    q = qkv[:, :n_heads * D].view(B, n_heads, D)
    k = qkv[:, n_heads * D:(n_heads + n_kv_heads) * D].view(B, n_kv_heads, D)
    v = qkv[:, (n_heads + n_kv_heads) * D:].view(B, n_kv_heads, D)
    q, k = _rope(q, pos, cfg.rope_theta), _rope(k, pos, cfg.rope_theta)
    for b in range(B):
        kc[b, :, int(pos[b])] = k[b]
        vc[b, :, int(pos[b])] = v[b]
    G = n_heads // n_kv_heads
    att = torch.empty((B, n_heads, D), device=x.device)
    for b in range(B):
        n = int(lens[b])
        kb = kc[b, :, :n].float().repeat_interleave(G, 0)            # [Hq, n, D]
        vb = vc[b, :, :n].float().repeat_interleave(G, 0)
        s = torch.einsum("hnd,hd->hn", kb, q[b]) / math.sqrt(D)
        p = torch.softmax(s.double(), -1).float()
        att[b] = torch.einsum("hn,hnd->hd", p, vb)
    if trace is not None:
        trace.update(q=q, k=k, v=v, att=att)
    o = att.view(B, n_heads * D) @ L["o"].float().T
    x = x + o if all_reduce is None else (x + o if rank == 0 else o)
    if all_reduce is not None:
        all_reduce(x)
    h = _rmsnorm(x, L["ln2"].float(), cfg.eps)
    gu = h @ L["gate_up"].float().T
    f = gu.shape[1] // 2
    a = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
    d = a @ L["down"].float().T
    x = x + d if all_reduce is None else (x + d if rank == 0 else d)
    if all_reduce is not None:
        all_reduce(x)
    return x
