"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py

It imports ``flatdecode`` from /root/reference/pkg/src (read-only; numba
backend), evaluates the hot-path functions on seeded inputs and writes:

  attention.npz  — batch_decode_attention (async/sync/reference) outputs,
                   _async_partials chunk states / violation indices, the
                   recompute mask and AttnStats, per case
  gemm.npz       — gemm_oracle, ImplA/B/C and flat_gemm outputs
  softmax.npz    — softmax_unified / partial_softmax_sync / check_bounds
  host.json      — integer/host logic: chunk_bounds, select_tile,
                   arithmetic_intensity, double_buffer_pipeline, calibrate,
                   _first_sustained, profile_shape(timers=...), dispatch,
                   save_table text

Inputs are fp16-representable float32 so the same fixtures can drive the
B200 kernels (fp16 storage) bit-identically on input.  Nothing on the GPU box
reads /root/reference; the fixtures are the committed pin.
"""

import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import flatdecode as fd  # noqa: E402
fda = sys.modules["flatdecode.attention"]
fdd = sys.modules["flatdecode.dispatch"]
fds = sys.modules["flatdecode.softmax"]

OUT = os.path.dirname(os.path.abspath(__file__))


def h(x):
    """Round to fp16 and back: fixtures are exactly representable in fp16."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def _stats(st):
    return np.array([st.rows_recomputed, st.rescale_ops, st.max_ops], dtype=np.int64)


def attention_cases():
    cases = []
    # 1-2: the paper's worked example (test_attention.py:95-143)
    V4 = h(np.random.default_rng(7).standard_normal((4, 4)))
    for logits in ([4.0, 5.0, 6.0, 7.0], [4.0, 5.0, 9.5, 7.0]):
        cases.append(dict(Q=h([logits]), K=np.eye(4, dtype=np.float32), V=V4, p=2,
                          scale=1.0, calib=(6.0, -3.0, 3.0)))
    # 3: chunk exp-sum overflow forces recompute (test_attention.py:147-159)
    V8 = h(np.random.default_rng(20).standard_normal((8, 8)))
    cases.append(dict(Q=h(np.full((1, 8), 87.0)), K=np.eye(8, dtype=np.float32), V=V8, p=1,
                      scale=1.0, calib=(0.0, -1.0, 87.9)))
    # 4: adversarial span +-40 (test_attention.py:78-87) — exercised in sync mode
    V8b = h(np.random.default_rng(5).standard_normal((8, 8)))
    cases.append(dict(Q=h([[40.0, -40.0, 20.0, -20.0, 0.0, 10.0, -10.0, 30.0]]),
                      K=np.eye(8, dtype=np.float32), V=V8b, p=4, scale=1.0,
                      calib=(0.0, -50.0, 50.0)))
    rng = np.random.default_rng(2026)

    def rand_case(M, L, d, p, scale, calib, inject=(), span=6.0, mult=3.0):
        # logits normalised to |x|<=span per row (test_acceptance.py:100-103), fp16 inputs
        K = h(rng.standard_normal((L, d)))
        V = h(rng.standard_normal((L, d)))
        Q = rng.standard_normal((M, d)).astype(np.float32)
        lg = scale * (Q.astype(np.float64) @ K.astype(np.float64).T)
        Q = Q * (span / np.abs(lg).max(axis=1, keepdims=True))
        for r in inject:
            Q[r] *= mult
        return dict(Q=h(Q), K=K, V=V, p=p, scale=scale, calib=calib)

    cases.append(rand_case(8, 64, 16, 4, 1.0, (0.0, -8.0, 8.0), inject=(2, 5)))
    cases.append(rand_case(16, 300, 64, 7, 1.0, (0.0, -8.0, 8.0), inject=(0, 9, 15)))
    cases.append(rand_case(3, 33, 8, 8, 1.0, (0.0, -8.0, 8.0)))
    cases.append(rand_case(1, 1, 8, 1, 1.0, (0.0, -8.0, 8.0)))
    # 9: Llama geometry slice: d=128, N(0,1) fp16 inputs, scale 1/sqrt(128),
    #    golden calibration -> no flags
    d = 128
    gold = fd.calibrate(np.random.default_rng(0).normal(0.0, 2.0, 1_000_000), 0.9999, 1.0)
    K = h(rng.standard_normal((512, d)))
    V = h(rng.standard_normal((512, d)))
    Q = h(rng.standard_normal((4, d)))
    cases.append(dict(Q=Q, K=K, V=V, p=4, scale=1.0 / math.sqrt(d),
                      calib=(gold.phi, gold.a, gold.b)))
    # 10: same geometry, two rows pushed far outside the band (x12, config 4 style)
    Q2 = Q.copy()
    Q2[1] = h(Q2[1] * 12.0)
    Q2[3] = h(Q2[3] * 12.0)
    cases.append(dict(Q=Q2, K=K, V=V, p=5, scale=1.0 / math.sqrt(d),
                      calib=(gold.phi, gold.a, gold.b)))
    return cases


def build_attention():
    out = {}
    cases = attention_cases()
    for i, c in enumerate(cases):
        calib = fd.ScalingCalibration(phi=c["calib"][0], a=c["calib"][1], b=c["calib"][2],
                                      coverage=1.0)
        cfg = fd.AttentionConfig(p=c["p"], scale=c["scale"], calib=calib)
        Q, K, V = c["Q"], c["K"], c["V"]
        pre = f"c{i}_"
        out[pre + "Q"], out[pre + "K"], out[pre + "V"] = Q, K, V
        out[pre + "meta"] = np.array([c["p"], c["scale"], *c["calib"]], dtype=np.float64)
        o_async, st_a = fd.batch_decode_attention(Q, K, V, cfg, "async")
        o_sync, st_s = fd.batch_decode_attention(Q, K, V, cfg, "sync")
        o_ref, _ = fd.batch_decode_attention(Q, K, V, cfg, "reference")
        Qp, Kp, Vp, bounds = fda._prep(Q, K, V, cfg)
        num, den, viol = fda._async_partials(Qp, Kp, Vp, cfg, bounds)
        out[pre + "out_async"] = o_async
        out[pre + "out_sync"] = o_sync
        out[pre + "out_ref"] = o_ref
        out[pre + "stats_async"] = _stats(st_a)
        out[pre + "stats_sync"] = _stats(st_s)
        out[pre + "num"] = num
        out[pre + "den"] = den
        out[pre + "viol"] = viol
        out[pre + "redo"] = (viol >= 0).any(axis=1)
        out[pre + "bounds"] = bounds
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **out)
    return len(cases)


def build_gemm():
    rng = np.random.default_rng(77)
    shapes = [(1, 256, 512), (3, 96, 40), (8, 128, 256), (17, 200, 136), (64, 256, 256),
              (7, 53, 101), (4, 640, 200)]
    out = {}
    for i, (m, n, k) in enumerate(shapes):
        a = h(rng.standard_normal((m, k)))
        b = h(rng.standard_normal((k, n)) / math.sqrt(k))
        pre = f"g{i}_"
        out[pre + "a"], out[pre + "b"] = a, b
        out[pre + "oracle"] = fd.gemm_oracle(a, b)
        out[pre + "implA"] = fd.impl_a_gemv(a, b)
        out[pre + "implB"] = fd.impl_b_flat(a, b, 8)
        out[pre + "implC"] = fd.impl_c_blocked(a, b)
        out[pre + "flat_16_32_db"] = fd.flat_gemm(a, b, fd.TileConfig(16, 32, double_buffer=True))
        out[pre + "flat_8_8"] = fd.flat_gemm(a, b, fd.TileConfig(8, 8))
    out["n_cases"] = np.array(len(shapes))
    np.savez_compressed(os.path.join(OUT, "gemm.npz"), **out)
    return len(shapes)


def build_softmax():
    rng = np.random.default_rng(31)
    out = {}
    vecs = [np.array([4, 5, 6, 7], np.float32), rng.uniform(-8, 8, 37).astype(np.float32),
            rng.uniform(-15, 15, 300).astype(np.float32), np.full(5, 3.25, np.float32)]
    for i, x in enumerate(vecs):
        out[f"s{i}_x"] = x
        out[f"s{i}_unified_phi0"] = fd.softmax_unified(x, 0.0)
        out[f"s{i}_unified_phi6"] = fd.softmax_unified(x, 6.0)
        for p in (1, 2, 4):
            if p <= x.size:
                out[f"s{i}_sync_p{p}"] = fd.partial_softmax_sync(x, p)
        out[f"s{i}_ref"] = fd.softmax_reference(x)
    out["n_cases"] = np.array(len(vecs))
    np.savez_compressed(os.path.join(OUT, "softmax.npz"), **out)


def build_host():
    g = {}
    g["chunk_bounds"] = [[n, p, fds.chunk_bounds(n, p).tolist()]
                         for n in (1, 7, 8, 33, 100, 1024, 32768) for p in (1, 2, 3, 4, 7, 64)
                         if p <= n]
    g["select_tile"] = []
    for (m, n, k) in [(8, 256, 4096), (8, 16384, 4096), (8, 8, 128), (1, 4096, 4096),
                      (8, 12288, 4096), (64, 11008, 4096), (4, 4096, 11008), (3, 48, 100),
                      (16, 512, 128)]:
        for w in (1, 8, 148):
            for tgt in (None, 32):
                t = fd.select_tile(fd.GemmShape(m, n, k), w, tgt)
                g["select_tile"].append([m, n, k, w, tgt, t.b_n, t.b_k, t.m_pad, t.double_buffer])
    g["arithmetic_intensity"] = []
    for (m, n, k) in [(8, 12288, 4096), (1, 4096, 4096), (64, 11008, 4096), (4, 1024, 512)]:
        for bn in (1, 8, 128, 1024):
            for bk in (8, 32, 64):
                e = fd.arithmetic_intensity(fd.GemmShape(m, n, k), bn, bk)
                g["arithmetic_intensity"].append([m, n, k, bn, bk, e.flops, e.bytes,
                                                  e.intensity, e.parallelism])
    g["double_buffer_pipeline"] = {str(T): fd.double_buffer_pipeline(T) for T in range(1, 14)}
    # calibration: the golden a1 plus small sample sets
    gold = fd.calibrate(np.random.default_rng(0).normal(0.0, 2.0, 1_000_000), 0.9999, 1.0)
    g["calibrate_golden"] = [gold.phi, gold.a, gold.b, gold.coverage]
    small = []
    rng = np.random.default_rng(9)
    for target in (0.6, 0.9, 0.999):
        s = rng.uniform(-30, 30, 57).astype(np.float32)
        c = fd.calibrate(s, target)
        small.append([s.tolist(), target, c.phi, c.a, c.b, c.coverage])
    c = fd.calibrate(np.full(1000, 2.5), 0.999, margin=1.0)
    small.append([[2.5] * 1000, 0.999, c.phi, c.a, c.b, c.coverage])
    g["calibrate_small"] = small
    # _first_sustained on random sequences
    fs = []
    rng = np.random.default_rng(4)
    for _ in range(200):
        n = int(rng.integers(2, 10))
        new = rng.uniform(0, 1, n).round(2).tolist()
        old = rng.uniform(0, 1, n).round(2).tolist()
        start = int(rng.integers(0, n))
        fs.append([new, old, start, fdd._first_sustained(new, old, start)])
    g["first_sustained"] = fs
    # profile_shape decision flow with injected medians (dispatch.py:316-317)
    ps = []
    sweeps = [(1, 2, 4, 8, 16, 32, 64, 128, 256), (1, 2, 4, 8, 16, 32, 64), (1, 4, 16)]
    for _ in range(150):
        sweep = sweeps[int(rng.integers(0, len(sweeps)))]
        med = {name: rng.uniform(0.1, 10.0, len(sweep)).round(3).tolist()
               for name in ("ImplA", "ImplB", "ImplC")}
        timers = {name: (lambda m, v=med[name], s=sweep: v[s.index(m)]) for name in med}
        e = fd.profile_shape(4096, 4096, m_sweep=sweep, timers=timers)
        ps.append([list(sweep), med["ImplA"], med["ImplB"], med["ImplC"], e.m1, e.m2])
    analytic = [({"ImplA": lambda m: 2.0 * m, "ImplB": lambda m: 10.0 + 0.5 * m,
                  "ImplC": lambda m: 100.0 + 0.1 * m}),
                ({"ImplA": lambda m: 1.0 * m, "ImplB": lambda m: 1e6 + m,
                  "ImplC": lambda m: 30.0 + 0.5 * m}),
                ({"ImplA": lambda m: 1.0, "ImplB": lambda m: 2.0, "ImplC": lambda m: 3.0})]
    for timers in analytic:
        sweep = sweeps[0]
        e = fd.profile_shape(64, 64, m_sweep=sweep, timers=timers)
        ps.append([list(sweep), [timers["ImplA"](m) for m in sweep],
                   [timers["ImplB"](m) for m in sweep], [timers["ImplC"](m) for m in sweep],
                   e.m1, e.m2])
    g["profile_decisions"] = ps
    # dispatch() over a grid
    t = fd.DispatchTable(fingerprint="golden")
    entries = [(12288, 4096, 4, 64), (4096, 4096, 8, 8), (11008, 4096, 2, 128),
               (4096, 11008, 1, 512)]
    for n, k, m1, m2 in entries:
        t.add(fd.DispatchEntry(n=n, k=k, m1=m1, m2=m2))
    g["dispatch_entries"] = entries
    g["dispatch_grid"] = [[m, n, k, fd.dispatch(m, n, k, t).value]
                          for (n, k, _, _) in entries for m in range(1, 300, 3)]
    path = "/tmp/golden_table.tbl"
    fd.save_table(t, path)
    g["table_text"] = open(path).read()
    with open(os.path.join(OUT, "host.json"), "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    assert fd.backend.active_backend() == "numba", "golden fixtures come from the numba backend"
    na = build_attention()
    ng = build_gemm()
    build_softmax()
    build_host()
    print(f"wrote {na} attention cases, {ng} gemm cases, softmax + host fixtures to {OUT}")
