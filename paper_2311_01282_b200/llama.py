"""Llama-family decode step on the three hot paths (the
reference's toy caller is pipeline.py:88-163).

One decode step for a batch of B sequences, all in libfdpp kernels:

    embed -> L x [ rmsnorm -> QKV GEMM -> RoPE + KV append -> async attention
                   (+ flagged-row recompute) -> O GEMM (+residual fused) ->
                   rmsnorm -> gate|up GEMM -> SiLU*up -> down GEMM (+residual) ]
          -> rmsnorm -> LM-head GEMM -> argmax -> advance positions

Every GEMM goes through the heuristic dispatch table (ImplA/B/C chosen per
[N, K] at M = B).  The whole step is captured once into a CUDA graph: the
attended lengths live in device memory (``seq_lens``) and advance on the
device, so replaying the same graph decodes successive tokens with no host
work between kernels.

Geometry is real Llama-2 (gate projection, RMSNorm, RoPE, residuals, LM
head), not the reference's 4-GEMM toy layer; weights are random-init
(N(0, 1/K)), the KV cache is prefilled with N(0, 1) synthetic state.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib, tp as _tp, workspace
from . import dispatch as _dispatch_mod  # noqa: F401  (module, not the function)
from .attention import AttentionConfig, decode_attention
from .gemm import (PackedWeight, interleave_gate_up, permute_gate_up_for_gemv, permute_qkv_for_gemv,
                   run_fused)
from .softmax import ScalingCalibration

import importlib

D = importlib.import_module("paper_2311_01282_b200.dispatch")

# calibrate(default_rng(0).normal(0, 2, 1e6), 0.9999, 1.0)
GOLDEN_CALIB = ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594,
                                  coverage=0.999989)


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    n_layers: int
    vocab: int
    rope_theta: float = 10000.0
    eps: float = 1e-5

    def gemm_shapes(self, tp: int = 1):
        """[N, K] of each dispatched GEMM in one step (on one of `tp` ranks)."""
        return _tp.rank_gemm_shapes(self, tp)

    def weight_bytes(self, dtype_bytes=2, tp: int = 1) -> int:
        """Bytes one rank streams per step (sharded projections + replicated
        embedding row reads are negligible; LM head replicated)."""
        per_layer = sum(n * k for n, k in list(self.gemm_shapes(tp).values())[:4]) + 2 * self.hidden
        return dtype_bytes * (self.n_layers * per_layer + 2 * self.vocab * self.hidden + self.hidden)

    def kv_bytes_per_token(self, dtype_bytes=2, tp: int = 1) -> int:
        return 2 * self.n_layers * (self.n_kv_heads // tp) * self.head_dim * dtype_bytes


LLAMA2_7B = LlamaConfig("llama2-7b", 4096, 32, 32, 128, 11008, 32, 32000)
LLAMA2_70B = LlamaConfig("llama2-70b", 8192, 64, 8, 128, 28672, 80, 32000)
CHATGLM2_6B = LlamaConfig("chatglm2-6b", 4096, 32, 2, 128, 13696, 28, 65024)


def build_dispatch_table(cfg: LlamaConfig, m_sweep=D.B200_M_SWEEP, reps=5, dtype=torch.float16,
                         fingerprint=None, tp: int = 1):
    """Profile every GEMM shape of a decode step on this device (profile_shape)."""
    table = D.DispatchTable(fingerprint=fingerprint or D.default_fingerprint())
    for n, k in sorted(set(cfg.gemm_shapes(tp).values())):
        table.add(D.profile_shape(n, k, m_sweep=m_sweep, reps=reps, dtype=dtype))
    return table


def fold_norm(pw: PackedWeight, norm_w) -> PackedWeight:
    """W'[n, k] = W[n, k] * w[k]: RMSNorm's weight folded into the next
    projection, so the GEMM consumes the raw residual stream and only scales
    each output row by its inverse RMS in the epilogue (fdpp_gemm_fuse x_op 3).
    All-ones weights (random init) return the same tensor."""
    if bool((norm_w == 1).all()):
        return pw
    w = pw.w.clone()
    w[:, : pw.K] = (w[:, : pw.K].float() * norm_w.float()[None, :]).to(w.dtype)
    return PackedWeight(w, pw.K, pw.N)


# the decode step lets attention stream K/V rows before its PDL wait (only the
# appended row comes from the QKV epilogue); FDPP_KV_PREFETCH=0 disables it (A/B)
KV_PREFETCH = os.environ.get("FDPP_KV_PREFETCH", "1") != "0"


class LlamaDecoder:
    """Random-init Llama decode engine over libfdpp (one replica per GPU)."""

    def __init__(self, cfg: LlamaConfig, batch: int, max_len: int, *, table=None,
                 calib: ScalingCalibration = GOLDEN_CALIB, dtype=torch.float16, seed: int = 0,
                 attn_p: int = 0, attn_splits: int = 0, n_layers: int = None, fused: bool = True,
                 tp_rank: int = 0, tp_size: int = 1, group=None, weights: dict = None,
                 collective: bool = True, gemv_step: bool = False, allreduce=None):
        """tp_size > 1: this process is rank tp_rank of a tensor-parallel group
        (tp.py): sharded QKV / O / gate|up / down, local heads and KV cache, one
        NCCL all-reduce of the residual stream after O and after down (captured
        in the step's CUDA graph).  weights: optional FULL model weights
        {"layers": [{qkv, o, gate_up, down ([N, K]), ln1, ln2}], "embed",
        "lm_head" ([vocab, hidden]), "ln_f"} to shard; default random init.
        allreduce: a ``PeerAllReduce`` (allreduce.py) for this rank: the O / down
        projections reduce across ranks inside their epilogue over peer memory
        (residual and next-RMSNorm sums of squares fused too) instead of the
        NCCL all-reduce + row-ssq kernel."""
        _lib.require_cuda()
        self.cfg, self.B, self.max_len, self.dtype = cfg, batch, max_len, dtype
        self.n_layers = n_layers or cfg.n_layers
        self.tp_rank, self.tp_size, self.group = tp_rank, tp_size, group
        # collective=False: one rank's shard alone on one GPU (per-GPU compute of a
        # t-way TP step; the all-reduce is omitted, the row-ssq kernel still runs)
        self.collective = collective
        self.allreduce = allreduce if tp_size > 1 else None
        sd = _tp.shard_dims(cfg, tp_size)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        g = torch.Generator(device=dev).manual_seed(seed + 7919 * tp_rank)   # sharded tensors
        g_rep = torch.Generator(device=dev).manual_seed(seed)                # replicated tensors
        shapes = cfg.gemm_shapes(tp_size)

        def w(n, k, gen=g):
            t = torch.empty((n, k), dtype=dtype, device=dev)
            t.normal_(0.0, 1.0 / math.sqrt(k), generator=gen)
            return PackedWeight(t, k, n)

        def packed(t):
            t = t.to(device=dev, dtype=dtype).contiguous()
            return PackedWeight(t, t.shape[1], t.shape[0])

        self.layers = []
        for li in range(self.n_layers):
            if weights is not None:
                Ls = _tp.shard_layer(weights["layers"][li], cfg, tp_rank, tp_size)
                self.layers.append({k: packed(Ls[k]) for k in ("qkv", "o", "gate_up", "down")} |
                                   {k: Ls[k].to(device=dev, dtype=dtype) for k in ("ln1", "ln2")})
                continue
            self.layers.append({
                "qkv": w(*shapes["qkv"]), "o": w(*shapes["o"]),
                "gate_up": w(*shapes["gate_up"]), "down": w(*shapes["down"]),
                "ln1": torch.ones(cfg.hidden, dtype=dtype, device=dev),
                "ln2": torch.ones(cfg.hidden, dtype=dtype, device=dev),
            })
        if weights is not None:
            self.embed = weights["embed"].to(device=dev, dtype=dtype).contiguous()
            self.lm_head = packed(weights["lm_head"])
            self.ln_f = weights["ln_f"].to(device=dev, dtype=dtype)
        else:
            self.embed = torch.empty((cfg.vocab, cfg.hidden), dtype=dtype, device=dev).normal_(
                0, 1, generator=g_rep)
            self.lm_head = w(*shapes["lm_head"], gen=g_rep)
            self.ln_f = torch.ones(cfg.hidden, dtype=dtype, device=dev)
        Hq, Hkv, Dh = sd.n_heads, sd.n_kv_heads, cfg.head_dim
        self.n_heads_local, self.n_kv_heads_local = Hq, Hkv
        self.k_cache = [torch.empty((batch, Hkv, max_len, Dh), dtype=dtype, device=dev)
                        for _ in range(self.n_layers)]
        self.v_cache = [torch.empty_like(self.k_cache[0]) for _ in range(self.n_layers)]
        B = batch
        self.x = torch.zeros((B, cfg.hidden), dtype=dtype, device=dev)
        self.h = torch.zeros_like(self.x)
        self.qkv = torch.zeros((B, shapes["qkv"][0]), dtype=dtype, device=dev)
        self.q = torch.zeros((B, Hq, Dh), dtype=dtype, device=dev)
        self.attn = torch.zeros((B, Hq, Dh), dtype=dtype, device=dev)
        self.ffn_local = sd.ffn
        self.gu = torch.zeros((B, 2 * sd.ffn), dtype=dtype, device=dev)
        self.act = torch.zeros((B, sd.ffn), dtype=dtype, device=dev)
        self.logits = torch.zeros((B, cfg.vocab), dtype=dtype, device=dev)
        self.ids = torch.zeros(B, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(B, dtype=torch.int32, device=dev)
        self.lens = torch.ones(B, dtype=torch.int32, device=dev)
        self.row_flags = torch.zeros((B, Hq), dtype=torch.uint8, device=dev)
        # fused step: per-(128-column tile, row) sums of squares of the residual
        # stream, written by the embed / O / down epilogues, read by the next
        # GEMM's RMSNorm prologue
        self.fused = fused
        nt = max(1, -(-cfg.hidden // 128))
        # sized for either producer: ImplB epilogues write hidden/128 tiles, the
        # fused GEMV one tile per 8 columns
        self.ssq_a = torch.zeros((max(nt, cfg.hidden // 8), B), dtype=torch.float32, device=dev)
        self.ssq_b = torch.zeros_like(self.ssq_a)
        self.ssq_tiles = nt
        self.recomputed = torch.zeros(1, dtype=torch.int32, device=dev)
        self.attn_cfg = AttentionConfig(p=attn_p or "auto", scale=1.0 / math.sqrt(Dh), calib=calib,
                                        splits_per_chunk=attn_splits)
        if table is None:
            table = build_dispatch_table(cfg, dtype=dtype, tp=tp_size)
        self.table = table
        # per-GEMM choice of the heuristic dispatch (the reference's decision flow)
        self.table_choices = {op: D.dispatch(B, n, k, table) for op, (n, k) in shapes.items()}
        # The fused step runs every projection on ImplB (its prologue/epilogue
        # fusions remove the RMSNorm / RoPE / SiLU / residual kernels).  The table
        # decides per GEMM; the step decides on the whole layer: at B = 1 the GEMV
        # wins each GEMM in isolation (tables/b200_decode.tbl) but the unfused step
        # is slower (profiles/r1_bench: 3.33 vs 2.80 ms).  ImplC (M beyond the
        # flat-GEMM band) still forces the unfused step.
        fused = fused and all(c != D.KernelChoice.IMPL_C for c in self.table_choices.values())
        # gemv_step (B <= 2, the table picking the GEMV for every projection): the
        # fused step on fdpp_gemv_fused.  Off by default: per GEMM it ties ImplB and
        # the B = 1 step measured 2.93 vs 2.83 ms on ImplB (the GEMV epilogues' scattered
        # RoPE / SiLU stores; profiles/r1_bench).
        self.step_impl = ("A" if gemv_step and fused and B <= 2 and all(
            c == D.KernelChoice.IMPL_A for c in self.table_choices.values()) else "B")
        if self.allreduce is not None:
            self.step_impl = "B"  # the fused all-reduce lives in the ImplB cluster epilogue
        self.gemv_ssq_tiles = cfg.hidden // 8
        kind = D.KernelChoice.IMPL_A if self.step_impl == "A" else D.KernelChoice.IMPL_B
        self.choices = ({op: kind for op in shapes} if fused else dict(self.table_choices))
        if tp_size > 1 and not fused:
            raise NotImplementedError("tensor parallelism runs on the fused (ImplB) decode step")
        self.graph = None
        self._host_pos = None    # host mirror of the decode position (prefill_random / rewind)
        self._layer_hook = None  # calibrate(): samples attention inputs after each QKV
        if fused:  # fold the RMSNorm weights into the following projections' columns
            for L in self.layers:
                if self.step_impl == "A":
                    L["qkv_f"] = permute_qkv_for_gemv(fold_norm(L["qkv"], L["ln1"]))
                    L["gate_up_f"] = permute_gate_up_for_gemv(fold_norm(L.pop("gate_up"), L["ln2"]))
                else:
                    L["qkv_f"] = fold_norm(L["qkv"], L["ln1"])
                    L["gate_up_f"] = interleave_gate_up(fold_norm(L.pop("gate_up"), L["ln2"]))
            self.lm_head_f = fold_norm(self.lm_head, self.ln_f)
        self.fused = fused
        self._tp_size = tp_size

    @property
    def launches_per_step(self) -> int:
        """Kernels one decode step launches: embed + L x (qkv+rope, attention (1
        launch when the cluster recomputes its own flagged rows, else 2), o,
        gate_up+silu, down [+ 2 row-ssq after the all-reduces]) + lm_head +
        argmax + advance (unfused: 8 + attention per layer, + 4)."""
        from .attention import launches
        na = launches(self.q, self.k_cache[0], self.attn_cfg, mode="async")
        if self.fused:
            per_layer = 4 + na + (2 if self._tp_size > 1 and self.allreduce is None else 0)
            return 1 + self.n_layers * per_layer + 3
        return 1 + self.n_layers * (8 + na) + 4

    # ------------------------------------------------------------------ calibration
    def calibrate(self, target_coverage: float = 0.9999, margin: float = 1.0, samples_per_layer: int = 65536,
                  seed: int = 0, apply: bool = True) -> ScalingCalibration:
        """Fit the unified phi and band to this model's logits:
        one eager decode step whose attention inputs (RoPE'd q, the KV cache with
        the new row) are sampled on the device after every layer's QKV projection
        (attention.sample_logits), then the reference's calibrate (softmax.py:219-266)
        on the host.  The step's state changes (positions, tokens, KV rows) are undone."""
        import numpy as np
        from .attention import sample_logits
        from .softmax import calibrate as _calibrate
        saved = (self.pos.clone(), self.lens.clone(), self.ids.clone())
        samples = []

        def hook(li):
            samples.append(sample_logits(self.q, self.k_cache[li], self.attn_cfg.scale, samples_per_layer,
                                         seq_lens=self.lens, seed=seed * 1000003 + li))
        self._layer_hook = hook
        try:
            self.enqueue_step()
        finally:
            self._layer_hook = None
        torch.cuda.synchronize()
        self.pos.copy_(saved[0])
        self.lens.copy_(saved[1])
        self.ids.copy_(saved[2])
        cal = _calibrate(torch.cat(samples).cpu().numpy().astype(np.float32), target_coverage, margin)
        if apply:
            self.attn_cfg = AttentionConfig(p=self.attn_cfg.p, scale=self.attn_cfg.scale, calib=cal,
                                            splits_per_chunk=self.attn_cfg.splits_per_chunk)
            self.graph = None  # the captured step holds the old calibration
        return cal

    # ------------------------------------------------------------------ state
    def prefill_random(self, L: int, seed: int = 1):
        """Synthetic prompt state: KV rows [0, L) ~ N(0, 1); next token at L."""
        if L + 1 > self.max_len:
            raise ValueError("prefill length exceeds the cache")
        g = torch.Generator(device=self.device).manual_seed(seed)
        for kc, vc in zip(self.k_cache, self.v_cache):
            kc[:, :, :L].normal_(0, 1, generator=g)
            vc[:, :, :L].normal_(0, 1, generator=g)
        self.pos.fill_(L)
        self.lens.fill_(L + 1)
        self.ids.random_(0, self.cfg.vocab, generator=g)
        self._host_pos = L

    def rewind(self, L: int):
        """Move every sequence back to position L (the next token is written at
        row L again); the KV rows [0, L) are kept."""
        if not 0 <= L < self.max_len:
            raise ValueError(f"position {L} outside the cache (max_len {self.max_len})")
        self.pos.fill_(L)
        self.lens.fill_(L + 1)
        self._host_pos = L

    @property
    def steps_left(self):
        """Decode steps the KV cache still has rows for (None: positions were set
        directly on the device and are not tracked on the host)."""
        return None if self._host_pos is None else self.max_len - self._host_pos

    # ------------------------------------------------------------------ one step
    def _gemm(self, op, a, pw, out, residual=None):
        D.run_device(self.choices[op], a, pw, out=out, residual=residual, ws_tag="decode_gemm")

    def enqueue_step(self):
        """Enqueue one decode step on the current stream (no host sync)."""
        if self.fused:
            return self._enqueue_fused()
        return self._enqueue_unfused()

    def _enqueue_fused(self):
        """Seven launches per layer.  RMSNorm is folded: its weight is
        pre-multiplied into the QKV / gate|up / LM-head weight columns and each
        output row is scaled by its inverse RMS in the GEMM epilogue, from the
        per-(tile, row) sums of squares the previous residual GEMM's epilogue
        (or the embedding) wrote.  RoPE + KV append run in the QKV epilogue, the
        residual adds in the O / down epilogues."""
        cfg, B, dt = self.cfg, self.B, _lib.dtype_code(self.dtype)
        lib = _lib.load()
        st = _lib.stream_handle()
        Hq, Dh = self.n_heads_local, cfg.head_dim
        ar = self.allreduce        # fused peer-memory all-reduce in the O / down epilogues
        tp = self.tp_size > 1 and ar is None  # separate NCCL all-reduce after O / down
        lead = self.tp_rank == 0 or ar is not None  # ranks whose epilogue adds the residual
        impl = self.step_impl      # "B": tcgen05 flat GEMM; "A": fused GEMV (B <= 2)
        # sums-of-squares tiles the residual GEMMs leave for the next folded RMSNorm
        res_tiles = 1 if tp else (self.gemv_ssq_tiles if impl == "A" else self.ssq_tiles)

        def all_reduce_x(ssq):
            # x = sum over ranks of (x + partial_0, partial_1, ...); then the
            # next projection's folded-RMSNorm input (one tile per row)
            import torch.distributed as dist
            if self.collective:
                dist.all_reduce(self.x, group=self.group)
            _lib.check(lib.fdpp_row_ssq(self.x.data_ptr(), ssq.data_ptr(), B, cfg.hidden, dt,
                                        _lib.stream_handle()), "row_ssq")

        _lib.check(lib.fdpp_embed(self.ids.data_ptr(), self.embed.data_ptr(), self.x.data_ptr(), B,
                                  cfg.hidden, self.ssq_a.data_ptr(), dt, st), "embed")
        ssq_tiles = 1
        for li, L in enumerate(self.layers):
            kc, vc = self.k_cache[li], self.v_cache[li]
            run_fused(self.x, L["qkv_f"], x_op=3, ssq_in=self.ssq_a, ssq_tiles=ssq_tiles,
                      eps=cfg.eps, ws_tag="decode_gemm", impl=impl,
                      rope={"q_out": self.q, "k_cache": kc, "v_cache": vc, "pos": self.pos,
                            "theta": cfg.rope_theta})
            if self._layer_hook is not None:
                self._layer_hook(li)
            # the QKV epilogue / rope_append just wrote only row pos of the caches
            decode_attention(self.q, kc, vc, self.attn_cfg, "async", out=self.attn,
                             seq_lens=self.lens, row_flags=self.row_flags, counter=self.recomputed,
                             kv_prefetch=KV_PREFETCH)
            run_fused(self.attn.view(B, Hq * Dh), L["o"], out=self.x, residual=self.x if lead else None,
                      ssq_out=None if tp or impl == "A" else self.ssq_b, ws_tag="decode_gemm", impl=impl,
                      allreduce=ar)
            if tp:
                all_reduce_x(self.ssq_b)  # (the fused GEMV re-derives the norm from x itself)
            run_fused(self.x, L["gate_up_f"], x_op=3, ssq_in=self.ssq_b, silu_out=self.act,
                      ssq_tiles=res_tiles, eps=cfg.eps, ws_tag="decode_gemm", impl=impl)
            run_fused(self.act, L["down"], out=self.x, residual=self.x if lead else None,
                      ssq_out=None if tp or impl == "A" else self.ssq_a, ws_tag="decode_gemm", impl=impl,
                      allreduce=ar)
            if tp:
                all_reduce_x(self.ssq_a)
            ssq_tiles = res_tiles
        run_fused(self.x, self.lm_head_f, out=self.logits, x_op=3, ssq_in=self.ssq_a,
                  ssq_tiles=ssq_tiles, eps=cfg.eps, ws_tag="decode_gemm", impl=impl)
        _lib.check(lib.fdpp_argmax(self.logits.data_ptr(), self.ids.data_ptr(), B, cfg.vocab, dt, st),
                   "argmax")
        _lib.check(lib.fdpp_advance_positions(self.pos.data_ptr(), self.lens.data_ptr(), B, st),
                   "advance")

    def _enqueue_unfused(self):
        cfg, B, dt = self.cfg, self.B, _lib.dtype_code(self.dtype)
        lib = _lib.load()
        st = _lib.stream_handle()
        Hq, Hkv, Dh = self.n_heads_local, self.n_kv_heads_local, cfg.head_dim
        _lib.check(lib.fdpp_embed(self.ids.data_ptr(), self.embed.data_ptr(), self.x.data_ptr(), B,
                                  cfg.hidden, None, dt, st), "embed")
        for li, L in enumerate(self.layers):
            _lib.check(lib.fdpp_rmsnorm(self.x.data_ptr(), L["ln1"].data_ptr(), self.h.data_ptr(), B,
                                        cfg.hidden, cfg.eps, dt, st), "rmsnorm")
            self._gemm("qkv", self.h, L["qkv"], self.qkv)
            kc, vc = self.k_cache[li], self.v_cache[li]
            _lib.check(lib.fdpp_rope_append(self.qkv.data_ptr(), self.q.data_ptr(), kc.data_ptr(),
                                            vc.data_ptr(), self.pos.data_ptr(), B, Hq, Hkv, Dh,
                                            kc.stride(0), kc.stride(1), cfg.rope_theta, dt, st),
                       "rope_append")
            if self._layer_hook is not None:
                self._layer_hook(li)
            # the QKV epilogue / rope_append just wrote only row pos of the caches
            decode_attention(self.q, kc, vc, self.attn_cfg, "async", out=self.attn,
                             seq_lens=self.lens, row_flags=self.row_flags, counter=self.recomputed,
                             kv_prefetch=KV_PREFETCH)
            self._gemm("o", self.attn.view(B, Hq * Dh), L["o"], self.x, residual=self.x)
            _lib.check(lib.fdpp_rmsnorm(self.x.data_ptr(), L["ln2"].data_ptr(), self.h.data_ptr(), B,
                                        cfg.hidden, cfg.eps, dt, st), "rmsnorm")
            self._gemm("gate_up", self.h, L["gate_up"], self.gu)
            _lib.check(lib.fdpp_silu_mul(self.gu.data_ptr(), self.act.data_ptr(), B, self.ffn_local, dt, st),
                       "silu_mul")
            self._gemm("down", self.act, L["down"], self.x, residual=self.x)
        _lib.check(lib.fdpp_rmsnorm(self.x.data_ptr(), self.ln_f.data_ptr(), self.h.data_ptr(), B,
                                    cfg.hidden, cfg.eps, dt, st), "rmsnorm")
        self._gemm("lm_head", self.h, self.lm_head, self.logits)
        _lib.check(lib.fdpp_argmax(self.logits.data_ptr(), self.ids.data_ptr(), B, cfg.vocab, dt, st),
                   "argmax")
        _lib.check(lib.fdpp_advance_positions(self.pos.data_ptr(), self.lens.data_ptr(), B, st),
                   "advance")

    def capture(self):
        """Capture one step into a CUDA graph (warms every kernel first)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            saved = (self.pos.clone(), self.lens.clone(), self.ids.clone())
            self.enqueue_step()                       # warm: attributes, tensor maps, workspaces
            self.pos.copy_(saved[0]); self.lens.copy_(saved[1]); self.ids.copy_(saved[2])
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.enqueue_step()
        torch.cuda.synchronize()
        self.graph = g
        return g

    def step(self):
        # every step appends one KV row at `pos`: refuse to run past the cache
        # (the append kernels also skip rows >= max_len, so nothing is corrupted)
        if self._host_pos is not None and self._host_pos >= self.max_len:
            raise RuntimeError(f"KV cache full: position {self._host_pos} >= max_len {self.max_len}; "
                               "rewind() or allocate a longer cache")
        if self.graph is None:
            self.capture()
        self.graph.replay()
        if self._host_pos is not None:
            self._host_pos += 1

    def decode(self, ids_host, out_host):
        """End-to-end step through the public API: H2D copy of this step's token
        ids (pinned host int32 [B]), one graph replay, D2H of the next ids."""
        self.ids.copy_(ids_host, non_blocking=True)
        self.step()
        out_host.copy_(self.ids, non_blocking=True)
        return out_host
