"""Benchmark: Llama-2-7B decode tokens/s on B200 through the three hot paths.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--kv-len L]
    python bench.py --impl reference ...        # the reference's CPU path (oracle port)

A "step" is one full decode step (32 layers, real Llama-2-7B geometry,
random-init fp16 weights, N(0,1) KV cache prefilled to L tokens) replayed from
one CUDA graph; per-GPU work is fixed as N grows (data-parallel replicas, no
collective: ``scaling`` = "weak").  The working set (13.2 GB weights + the KV
cache) is ~100x the 126 MB L2, so every step streams from HBM.

Printed JSON line (rank 0): value = device-timed tokens/s (max over ranks),
e2e = the same metric through the public API (LlamaDecoder.decode: pinned H2D
of the step's token ids, graph replay, D2H of the next ids, every step),
roofline = the dominant kernel's achieved HBM GB/s from CUDA events on its own
launches (per-op graph over all layers), cpu_baseline = the oracle port on
this host's cores (rank 0, N=1).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Llama-2-7B decode tokens/s at 1/8 GPU; attn+flat-GEMM HBM GB/s vs 8 TB/s"
UNIT = "tokens/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(int(r[0]) for r in rows)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------- CPU leg
def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class CpuReference:
    """The reference's CPU path for one decode step of this workload, restated
    by the oracle's C port of its numba kernels (kind "port"): every decoder
    layer runs its four projections through ImplA -- the kernel the
    reference's own dispatch picks on CPU at every M <= 64 --
    and async unified-phi attention (p = 4, pipeline.py:100-101) once per
    (batch, kv-head) with the G query rows sharing that K/V
    (pipeline.py:121-135); the LM head is one more ImplA GEMM.

    A full step is minutes of CPU work, so the timed unit is ONE decoder layer
    (all of its GEMMs and all of its attention calls, nothing sampled inside
    it): step time = n_layers x the median layer + the LM head (timed once).
    The K/V of the B x Hkv calls rotate over `n_kv` distinct 1-head caches
    (> the host's L3, so every call streams its K/V from DRAM like the
    reference's per-sequence caches)."""

    def __init__(self, B, L, cfg, threads=None, n_kv=64, seed=0):
        import numpy as np
        from oracle import flatdecode_oracle as O
        self.O, self.np = O, np
        self.cores = O.set_threads(threads or os.cpu_count() or 1)
        self.B, self.L, self.cfg = B, L, cfg
        rng = np.random.default_rng(seed)
        self.shapes = cfg.gemm_shapes()
        self.w = {op: rng.standard_normal((k, n), dtype=np.float32) / np.float32(k ** 0.5)
                  for op, (n, k) in self.shapes.items() if op != "lm_head"}
        self.x = {op: rng.standard_normal((B, k), dtype=np.float32) for op, (n, k) in self.shapes.items()}
        self.G = cfg.n_heads // cfg.n_kv_heads
        Dh = cfg.head_dim
        self.n_kv = n_kv
        self.kv = [(rng.standard_normal((L, Dh), dtype=np.float32),
                    rng.standard_normal((L, Dh), dtype=np.float32)) for _ in range(n_kv)]
        self.q = rng.standard_normal((self.G, Dh), dtype=np.float32)
        self.calib = O.Calib(-7.775933742523193, -1.0, 16.577659606933594)
        self.scale = 1 / math.sqrt(Dh)
        self.t_head = None

    def layer(self):
        """Seconds for one decoder layer's reference work."""
        O = self.O
        t0 = time.perf_counter()
        for op in ("qkv", "o", "gate_up", "down"):
            O.impl_a_gemv(self.x[op], self.w[op])
        i = 0
        for _b in range(self.B):
            for _h in range(self.cfg.n_kv_heads):
                K, V = self.kv[i % self.n_kv]
                O.batch_decode_attention(self.q, K, V, 4, self.scale, self.calib, "async")
                i += 1
        return time.perf_counter() - t0

    def lm_head(self):
        if self.t_head is None:
            n, k = self.shapes["lm_head"]
            b = self.np.random.default_rng(1).standard_normal((k, n), dtype=self.np.float32)
            t0 = time.perf_counter()
            self.O.impl_a_gemv(self.x["lm_head"], b)
            self.t_head = time.perf_counter() - t0
        return self.t_head

    def step_seconds(self, layer_times):
        import statistics
        return self.cfg.n_layers * statistics.median(layer_times) + self.lm_head()

    def describe(self, n_layers_timed):
        return (f"timed unit = one full decoder layer at B={self.B}, L={self.L} (4 ImplA GEMMs on "
                f"the full weights + {self.B * self.cfg.n_kv_heads} async attention calls, G={self.G} "
                f"rows each, p=4); step = {self.cfg.n_layers} x median of {n_layers_timed} layers + the "
                f"LM head GEMM (timed once): extrapolation factor {self.cfg.n_layers} on the layer; "
                f"oracle C port of the reference's numba kernels, {self.cores} threads")


def cpu_reference_step(B, L, cfg, n_layers_timed=3):
    """cpu_baseline of the GPU arm: a bounded sample (a few layers, ~10-30 s)."""
    ref = CpuReference(B, L, cfg)
    ref.lm_head()
    times = [ref.layer() for _ in range(n_layers_timed)]
    return ref.step_seconds(times), ref.describe(n_layers_timed), ref.cores


# --------------------------------------------------------------------------- GPU leg
def _op_graph_time(torch, fn, reps):
    """Average device time of the launches enqueued by fn (captured as one
    graph, replayed reps times between CUDA events on the replay stream)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


MODELS = {"llama2-7b": "LLAMA2_7B", "chatglm2-6b": "CHATGLM2_6B", "llama2-70b": "LLAMA2_70B"}


def _load_table(D, cfg, tp):
    """The committed B200 dispatch table (tools/make_table.py); shapes it lacks
    get the measured B200 policy for M <= 64 (ImplB from M = 1, ImplC beyond:
    every profiled Llama shape, tables/b200_decode.medians.json)."""
    table = None
    for name in ("b200_decode.tbl", "b200_llama2_7b.tbl"):
        path = os.path.join(ROOT, "tables", name)
        if os.path.exists(path):
            table = D.load_table(path)
            break
    if table is None:
        table = D.DispatchTable(fingerprint=D.default_fingerprint())
    for n, k in cfg.gemm_shapes(tp).values():
        if (n, k) not in table.entries:
            table.add(D.DispatchEntry(n=n, k=k, m1=1, m2=128))
    return table


def _rotating_graph_time(torch, fns, reps=5):
    """Device seconds per call of a list of launch closures (one CUDA graph
    holding them all, replayed reps times): operands rotate so the working set
    exceeds L2."""
    t = _op_graph_time(torch, lambda: [f() for f in fns], reps)
    return t / len(fns)


def config1_attention_op(torch, fd, peak):
    """configs[0]: async decode attention op alone, B=1, 32 heads x 128, L=1024,
    fp16, N(0,1) inputs, golden calibration; in-graph over 8 rotating caches."""
    B, H, L, Dh = 1, 32, 1024, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
    cfg = fd.AttentionConfig.auto(1 / math.sqrt(Dh), cal)
    q = torch.randn((B, H, Dh), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    kvs = [(torch.randn((B, H, L, Dh), generator=g, device="cuda").half(),
            torch.randn((B, H, L, Dh), generator=g, device="cuda").half()) for _ in range(8)]
    # as in the decode step: the preceding kernel wrote no K/V row (kv_prefetch)
    fns = [lambda k=k, v=v: fd.decode_attention(q, k, v, cfg, "async", out=out, kv_prefetch=True)
           for k, v in kvs]
    t = _rotating_graph_time(torch, fns)
    byt = 2 * B * H * L * Dh * 2 + 2 * B * H * Dh * 2
    return {"us": round(t * 1e6, 2), "bytes": byt, "gbs": round(byt / t / 1e9, 1),
            "frac": round(byt / t / 1e9 / peak, 3), "plan": list(fd.attention.plan(q, kvs[0][0], cfg)),
            "launches_per_call": fd.attention.launches(q, kvs[0][0], cfg),
            "note": "one cluster launch per call (flagged rows recomputed inside the cluster); 16.8 MB "
                    "moves in ~2.6 us at HBM speed, so launch/ramp latency dominates at this size"}


def config2_gemm_sweep(torch, fd, D, table, peak):
    """configs[1]: flat GEMM + dispatch over M in {1..64} x the Llama-2-7B
    projection shapes; in-graph, rotating weights (> L2)."""
    res = {}
    for n, k in ((12288, 4096), (4096, 4096), (11008, 4096), (4096, 11008)):
        nrot = max(4, min(16, int(1.2e9 // (n * k * 2))))
        ws = [fd.PackedWeight((torch.randn((n, k), device="cuda") / k ** 0.5).half(), k, n)
              for _ in range(nrot)]
        row = {}
        for m in (1, 2, 4, 8, 16, 32, 64):
            a = torch.randn((m, k), device="cuda").half()
            out = torch.empty((m, n), device="cuda", dtype=torch.half)
            ch = D.dispatch(m, n, k, table)
            t = _rotating_graph_time(torch, [lambda w=w: D.run_device(ch, a, w, out=out) for w in ws])
            byt = n * k * 2 + m * k * 2 + m * n * 2
            row[str(m)] = {"choice": ch.value, "us": round(t * 1e6, 2), "gbs": round(byt / t / 1e9, 1),
                           "frac": round(byt / t / 1e9 / peak, 3)}
        res[f"{n}x{k}"] = row
        del ws
    return res


def dispatch_report(D, table):
    """dispatch has no roofline -- its host cost (done once per M
    bucket at graph capture) and the reference's self-consistency criterion
    (test_acceptance.py:187-195) on the committed B200 profile."""
    path = os.path.join(ROOT, "tables", "b200_decode.medians.json")
    with open(path) as f:
        details = json.load(f)
    ref = D.load_table(os.path.join(ROOT, "tables", "b200_decode.tbl"))
    worst, bad = D.dispatch_regret(ref, details)
    reps = 20000
    t0 = time.perf_counter()
    for i in range(reps):
        D.dispatch(1 + (i & 63), 12288, 4096, table)
    host_ns = (time.perf_counter() - t0) / reps * 1e9
    return {"host_ns_per_call": round(host_ns, 1), "profile_points": sum(len(r) for r in details.values()),
            "max_dispatched_over_best": round(worst, 4), "points_over_1.10x": len(bad),
            "table": "tables/b200_decode.tbl (tools/make_table.py, profile_shape flow to M = 256)"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        # NCCL's init lines (communicator size per rank) make the N-rank launch observable
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if rank == 0:
            print(f"bench: {world} ranks over NCCL (one process per GPU)", file=sys.stderr, flush=True)
    else:
        torch.cuda.set_device(0)
    import paper_2311_01282_b200 as fd
    from paper_2311_01282_b200 import llama
    from paper_2311_01282_b200.attention import decode_attention
    import importlib
    D = importlib.import_module("paper_2311_01282_b200.dispatch")

    cfg = getattr(llama, MODELS[args.model])
    # tensor parallelism: --tp T over the launched ranks (dp = world / T groups);
    # --tp-shard T on one process: rank 0's shard alone, all-reduce omitted
    tp = args.tp if args.tp > 1 else 1
    shard_only = args.tp_shard > 1 and world == 1
    if shard_only:
        tp = args.tp_shard
    if world % (1 if shard_only else tp):
        raise SystemExit(f"--tp {tp} must divide the world size {world}")
    dp = world // (1 if shard_only else tp)
    tp_rank = 0 if shard_only else rank % tp
    group = None
    if tp > 1 and not shard_only:
        groups = [dist.new_group(list(range(d * tp, (d + 1) * tp))) for d in range(dp)]
        group = groups[rank // tp]
    B, L, K, W = args.batch, args.kv_len, args.steps, args.warmup
    table = _load_table(D, cfg, tp)
    ar = None
    if args.ar == "fused" and tp > 1 and not shard_only:
        # the O / down projections reduce across the TP group inside their GEMM
        # epilogue over IPC-mapped peer memory (allreduce.py) instead of NCCL
        from paper_2311_01282_b200.allreduce import PeerAllReduce
        ar = PeerAllReduce.create(group, cap=B * cfg.hidden)
    dec = llama.LlamaDecoder(cfg, B, L + max(K, W) + 16, table=table, seed=1000 + rank // tp,
                             tp_rank=tp_rank, tp_size=tp, group=group, collective=not shard_only,
                             allreduce=ar, gemv_step=args.gemv_step)
    dec.prefill_random(L, seed=2000 + rank // tp)
    if args.inject:
        # configs[3]: force the synchronized-softmax recompute: one key far
        # outside the calibrated band in `inject` (batch, kv-head) groups of
        # every layer flags all G query rows of those groups
        for kc in dec.k_cache:
            for r in range(args.inject):
                b, h = r % B, (r // B) % dec.n_kv_heads_local
                kc[b, h, L // 2].mul_(40.0)
    cal = None
    if args.calibrate:
        # fit phi / the band to this model's own logits (device-sampled after every
        # layer's QKV, then the reference's calibrate).  Off by default: at
        # coverage 0.9999 of single logits ~10% of 1K-key rows hold one outlier
        # and recompute (measured 9593 vs 3071 recomputed rows, 6.16 vs 5.97 ms)
        cal = dec.calibrate(target_coverage=args.calibrate, margin=1.0, samples_per_layer=32768)
    dec.capture()
    for _ in range(W):
        dec.step()
    # each timed loop decodes positions L .. L+K-1 (the cache holds L + max(K, W) + 16 rows)
    dec.rewind(L)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dev = torch.cuda.current_device()
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            dec.step()
        e1.record()
        e1.synchronize()
        torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        dist.barrier()
        t = torch.tensor([secs], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t.item())
    value = dp * B * K / secs          # tokens: each TP group decodes one batch
    ms_per_step = secs / K * 1e3
    recomputed = int(dec.recomputed.item())

    # ---- e2e through the public API (pinned host ids in, next ids out, every step)
    ids_h = torch.zeros(B, dtype=torch.int32).pin_memory()
    out_h = torch.zeros(B, dtype=torch.int32).pin_memory()
    ids_h.copy_(dec.ids.cpu())
    dec.rewind(L)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    e0.record()
    for _ in range(K):
        dec.decode(ids_h, out_h)      # H2D ids -> graph replay -> D2H next ids
        stream.synchronize()          # the host needs the tokens before the next step
        ids_h.copy_(out_h)
    e1.record()
    e1.synchronize()
    e2e_secs = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        t = torch.tensor([e2e_secs], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_secs = float(t.item())
    e2e_value = dp * B * K / e2e_secs

    # ---- per-op device time over all layers (roofline of the dominant kernel),
    # at the first timed position (attended length L + 1)
    dec.rewind(L)
    reps = 3
    hq, dh, hkv = dec.n_heads_local, cfg.head_dim, dec.n_kv_heads_local
    ops = {}

    def attn_all():
        for li in range(dec.n_layers):
            decode_attention(dec.q, dec.k_cache[li], dec.v_cache[li], dec.attn_cfg, "async",
                             out=dec.attn, seq_lens=dec.lens, row_flags=dec.row_flags,
                             counter=dec.recomputed, kv_prefetch=True)
    t_attn = _op_graph_time(torch, attn_all, reps) / dec.n_layers
    Lnow = min(int(dec.lens[0].item()), dec.max_len)   # keys the kernel attends
    attn_bytes = B * hkv * Lnow * dh * 2 * 2 + 2 * B * hq * dh * 2
    ops["attention_async(+recompute)"] = {"s_per_launch": t_attn, "bytes": attn_bytes,
                                          "launches_per_step": dec.n_layers}
    shapes = cfg.gemm_shapes(tp)
    from paper_2311_01282_b200.gemm import run_fused
    gb = lambda n, k: n * k * 2 + B * k * 2 + B * n * 2  # noqa: E731
    if dec.fused:
        L0 = dec.layers
        st = 1 if tp > 1 else (dec.gemv_ssq_tiles if dec.step_impl == "A" else dec.ssq_tiles)
        im = dec.step_impl
        per_op = {
            f"gemm_qkv+rmsnorm+rope[{shapes['qkv'][0]}x{shapes['qkv'][1]}]:Impl{im}": (
                lambda: [run_fused(dec.x, Ld["qkv_f"], x_op=3, ssq_in=dec.ssq_a, ssq_tiles=st,
                                   eps=cfg.eps, ws_tag="decode_gemm", impl=im,
                                   rope={"q_out": dec.q, "k_cache": dec.k_cache[i],
                                         "v_cache": dec.v_cache[i], "pos": dec.pos,
                                         "theta": cfg.rope_theta}) for i, Ld in enumerate(L0)],
                gb(*shapes["qkv"]), len(L0)),
            f"gemm_o+residual+ssq[{shapes['o'][0]}x{shapes['o'][1]}]:Impl{im}": (
                lambda: [run_fused(dec.attn.view(B, hq * dh), Ld["o"], out=dec.h, residual=dec.x,
                                   ssq_out=None if tp > 1 else dec.ssq_b, ws_tag="decode_gemm", impl=im)
                         for Ld in L0],
                gb(*shapes["o"]), len(L0)),
            f"gemm_gate_up+rmsnorm+silu[{shapes['gate_up'][0]}x{shapes['gate_up'][1]}]:Impl{im}": (
                lambda: [run_fused(dec.x, Ld["gate_up_f"], silu_out=dec.act, x_op=3, ssq_in=dec.ssq_b,
                                   ssq_tiles=st, eps=cfg.eps, ws_tag="decode_gemm", impl=im)
                         for Ld in L0],
                gb(*shapes["gate_up"]), len(L0)),
            f"gemm_down+residual+ssq[{shapes['down'][0]}x{shapes['down'][1]}]:Impl{im}": (
                lambda: [run_fused(dec.act, Ld["down"], out=dec.h, residual=dec.x,
                                   ssq_out=None if tp > 1 else dec.ssq_a, ws_tag="decode_gemm", impl=im)
                         for Ld in L0],
                gb(*shapes["down"]), len(L0)),
            f"gemm_lm_head+rmsnorm[{shapes['lm_head'][0]}x{shapes['lm_head'][1]}]:Impl{im}": (
                lambda: run_fused(dec.x, dec.lm_head_f, out=dec.logits, x_op=3, ssq_in=dec.ssq_a,
                                  ssq_tiles=st, eps=cfg.eps, ws_tag="decode_gemm", impl=im),
                gb(*shapes["lm_head"]), 1),
        }
    else:
        bufs = {"qkv": (dec.h, dec.qkv), "o": (dec.attn.view(B, hq * dh), dec.h),
                "gate_up": (dec.h, dec.gu), "down": (dec.act, dec.h), "lm_head": (dec.h, dec.logits)}
        per_op = {}
        for op in ("qkv", "o", "gate_up", "down", "lm_head"):
            a, out = bufs[op]
            ws = [Ld[op] for Ld in dec.layers] if op != "lm_head" else [dec.lm_head]
            ch = dec.choices[op]
            n, k = shapes[op]
            per_op[f"gemm_{op}[{n}x{k}]:{ch.value}"] = (
                lambda a=a, out=out, ws=ws, ch=ch: [D.run_device(ch, a, w, out=out, ws_tag="decode_gemm")
                                                    for w in ws], gb(n, k), len(ws))
    for name, (fn, byt, nl) in per_op.items():
        t = _op_graph_time(torch, fn, reps) / nl
        ops[name] = {"s_per_launch": t, "bytes": byt, "launches_per_step": nl}
    peak, peak_kind = _peaks()
    for name, o in ops.items():
        o["gbs"] = o["bytes"] / o["s_per_launch"] / 1e9
        o["share_of_step"] = o["s_per_launch"] * o["launches_per_step"] / (secs / K)
    dom_name = max(ops, key=lambda n: ops[n]["s_per_launch"] * ops[n]["launches_per_step"])
    dom = ops[dom_name]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            key = dom_name.split("[")[0].split(":")[0]
            traffic = tr.get(f"{args.model}/B{B}/L{L}", {}).get(key)
        except Exception:
            traffic = None
    # KV bytes at the mean attended length of the timed steps (L + 1 .. L + K)
    L_mean = L + (K + 1) / 2
    step_bytes = int(cfg.weight_bytes(tp=tp) + B * L_mean * cfg.kv_bytes_per_token(tp=tp))
    default_run = args.model == "llama2-7b" and tp == 1
    workload = {"llama2-7b": "llama2-7b decode step (configs[2])",
                "chatglm2-6b": "chatglm2-6b MQA decode step (configs[3])",
                "llama2-70b": "llama2-70b GQA decode step (configs[4])"}[args.model]
    par = f"dp{dp}" + (f"xtp{tp}" if tp > 1 and not shard_only else "")
    if tp > 1 and not shard_only:
        par += " (all-reduce: " + ("fused into the O/down epilogues, peer memory" if ar is not None else "NCCL") + ")"
    if shard_only:
        par = f"one tp{tp} shard on 1 GPU (all-reduce omitted)"
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": workload, "model": f"{cfg.name} geometry, random-init",
                   "layer": "Llama-style layer (gate GEMM, RMSNorm, RoPE, residual, LM head)",
                   "global_batch": dp * B, "batch_per_gpu": B, "kv_len": L, "parallelism": par,
                   "l2": f"inputs larger than L2 ({cfg.weight_bytes(tp=tp) / 1e9:.1f} GB weights + KV per step)",
                   "attention": f"async unified-phi, p={dec.attn_cfg.p}"
                                + (", GQA/MQA on tensor cores" if cfg.n_heads // cfg.n_kv_heads >= 4 else ""),
                   "gemm_choices": {op: c.value for op, c in dec.choices.items()},
                   "dispatch_table_choices": {op: c.value for op, c in dec.table_choices.items()},
                   "injected_groups_per_layer": args.inject,
                   "calibration": ("golden (SURVEY a1)" if cal is None else
                                   {"phi": round(cal.phi, 4), "a": round(cal.a, 4), "b": round(cal.b, 4),
                                    "coverage": round(cal.coverage, 6),
                                    "source": "LlamaDecoder.calibrate on this model's logits"})},
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": B * 4,
                "d2h_bytes_per_step": B * 4},
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": round(dom["gbs"], 1),
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(dom["gbs"] / peak, 4), "frac_of_8tbs": round(dom["gbs"] / 8000, 4),
                     "traffic": traffic, "bytes_per_launch": dom["bytes"],
                     "us_per_launch": round(dom["s_per_launch"] * 1e6, 2),
                     # attention bytes and time at the first timed position (L + 1 keys)
                     "kv_len_at_measure": Lnow},
        "step_hbm": {"bytes": step_bytes, "achieved_gbs": round(step_bytes / (secs / K) / 1e9, 1),
                     "frac": round(step_bytes / (secs / K) / 1e9 / peak, 4)},
        "kernels": {n: {"us": round(o["s_per_launch"] * 1e6, 2), "gbs": round(o["gbs"], 1),
                        "frac": round(o["gbs"] / peak, 3), "share": round(o["share_of_step"], 3)}
                    for n, o in ops.items()},
        "gpu_launches": K * dec.launches_per_step,
        "rows_recomputed": recomputed,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and default_run and not args.no_extras:
        line["configs"] = {"c1_attention_op_b1_l1024": config1_attention_op(torch, fd, peak),
                           "c2_gemm_dispatch_sweep": config2_gemm_sweep(torch, fd, D, table, peak),
                           "c2_dispatch": dispatch_report(D, table)}
    if rank == 0 and world == 1 and not args.no_cpu:
        t_step, desc, cores = cpu_reference_step(B, L, cfg)
        line["cpu_baseline"] = {"value": round(B / t_step, 4), "unit": UNIT, "cores": cores,
                                "kind": "port", "sample": desc, "cpu_model": _cpu_model(),
                                "extrapolation_factor": cfg.n_layers}
    if world > 1:
        dist.barrier()
        if ar is not None:
            ar.close()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2311_01282_b200 import llama  # config only (no GPU work)
    cfg = getattr(llama, MODELS[args.model])
    B, L = args.batch, args.kv_len
    ref = CpuReference(B, L, cfg)
    # W warm-up layers (page-in, thread pool) and the LM head, untimed; the
    # timed steps are K full decoder layers, each the unit described above
    for _ in range(max(1, args.warmup)):
        ref.layer()
    ref.lm_head()
    times = [ref.layer() for _ in range(args.steps)]
    t_step = ref.step_seconds(times)
    timed = sum(times)
    value = B / t_step
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(1, args.warmup), "ms_per_step": round(timed / args.steps * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.model} decode step (configs[2])", "model": f"{cfg.name} geometry, random-init",
                   "global_batch": B, "batch_per_gpu": B, "kv_len": L,
                   "parallelism": f"host CPU, {ref.cores} threads (reference numba path, restated in C)",
                   "step": "ms_per_step is the measured time of one timed unit (one full decoder layer); "
                           f"value = B / ({cfg.n_layers} x median layer + LM head)",
                   "extrapolation_factor": cfg.n_layers,
                   "ms_per_full_step": round(t_step * 1e3, 1),
                   "timed_seconds": round(timed, 2), "cpu_model": _cpu_model()},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": ref.cores, "kind": "port",
                         "sample": ref.describe(args.steps), "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _relaunch_distributed(args):
    """--gpus N > 1 without a torchrun environment: launch N ranks (one per
    GPU) under torch.distributed.run ourselves and return its exit code."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--kv-len", type=int, default=1024)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the configs[0]/[1] sub-benchmarks")
    ap.add_argument("--model", default="llama2-7b", choices=sorted(MODELS))
    ap.add_argument("--tp", type=int, default=1, help="tensor-parallel ranks per replica (torchrun)")
    ap.add_argument("--ar", default="nccl", choices=("nccl", "fused"),
                    help="TP all-reduce: NCCL after the O/down GEMMs, or fused into their epilogues")
    ap.add_argument("--tp-shard", type=int, default=1,
                    help="single GPU: run rank 0's shard of a T-way TP step (all-reduce omitted)")
    ap.add_argument("--gemv-step", action="store_true",
                    help="B <= 2: run the fused step on the CUDA-core GEMV (fdpp_gemv_fused) instead of ImplB")
    ap.add_argument("--calibrate", type=float, default=0.0,
                    help="calibrate phi/band on the model's logits at this coverage (default: SURVEY a1's golden calibration)")
    ap.add_argument("--inject", type=int, default=0,
                    help="(batch, kv-head) groups per layer forced through the recompute path")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
