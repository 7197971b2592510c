"""TEST INFRASTRUCTURE (runs only where /root/reference exists, i.e. the build
container, never on the GPU box): time the REAL reference (flatdecode, numba
backend, the reference's own timing.measure / median_mad) and this oracle's C
port side by side on the same host, same threads, same inputs -- the
calibration behind using the port as bench.py's cpu_baseline and reference arm
(BASELINE.md §3).  GEMMs time ImplA / ImplB / ImplC (the reference's
dispatch.py:73-145) and report the reference-dispatched choice (ImplA at every
M <= 64 on CPU) and the best of the three.

    python oracle/port_timing_calibration.py [--threads N]  -> profiles/r2/cpu_port_calibration.json
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_SRC = "/root/reference/pkg/src"


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _median(fn, reps, warmup=1):
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    if not os.path.isdir(REF_SRC):
        raise SystemExit("needs the reference sources (build container only)")
    os.environ["FLATDECODE_WORKERS"] = str(args.threads)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    import flatdecode as ref
    import importlib
    rd = importlib.import_module("flatdecode.dispatch")
    from flatdecode.timing import measure, median_mad
    import numba
    cores = args.threads
    out = {"host": _cpu_model(), "cpu_count": os.cpu_count(), "threads": cores,
           "numba": numba.__version__, "numba_threads": numba.get_num_threads(),
           "backend": ref.active_backend() if hasattr(ref, "active_backend") else "numba",
           "order": "every reference timing first, then the port (its thread pool would compete)",
           "ops": []}
    rng = np.random.default_rng(0)
    L, D, p = 1024, 128, 4
    scale = 1 / math.sqrt(D)
    calib_r = ref.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
    att = [(G, rng.standard_normal((G, D), dtype=np.float32), rng.standard_normal((L, D), dtype=np.float32),
            rng.standard_normal((L, D), dtype=np.float32)) for G in (1, 16)]
    gem = []
    for n, k in ((4096, 4096), (12288, 4096)):
        b = rng.standard_normal((k, n), dtype=np.float32) / np.float32(math.sqrt(k))
        for m in (1, 8, 32):
            gem.append((n, k, m, rng.standard_normal((m, k), dtype=np.float32), b))
    # ---- pass 1: the real reference (attention per head: its API is per head)
    cfg = ref.AttentionConfig(p=p, scale=scale, calib=calib_r)
    for G, Q, K, V in att:
        t_ref, _ = median_mad(measure(lambda: ref.batch_decode_attention(Q, K, V, cfg, "async"), reps=args.reps))
        out["ops"].append({"op": "batch_decode_attention async", "rows": G, "L": L, "D": D, "p": p, "reference_s": t_ref})
    for n, k, m, a_, b in gem:
        row = {"op": "gemm", "n": n, "k": k, "m": m}
        for name, fr in (("ImplA", lambda: rd.impl_a_gemv(a_, b)), ("ImplB", lambda: rd.impl_b_flat(a_, b, cores)),
                         ("ImplC", lambda: rd.impl_c_blocked(a_, b))):
            row[f"{name}_reference_s"], _ = median_mad(measure(fr, reps=args.reps))
        row["reference_best_of_three"] = min(("ImplA", "ImplB", "ImplC"), key=lambda nm: row[f"{nm}_reference_s"])
        row["reference_dispatched"] = "ImplA"
        out["ops"].append(row)
    # ---- pass 2: the oracle's C port, same inputs and thread count
    from oracle import flatdecode_oracle as O
    O.set_threads(cores)
    calib_o = O.Calib(-7.775933742523193, -1.0, 16.577659606933594)
    i = 0
    for G, Q, K, V in att:
        r = out["ops"][i]
        r["port_s"] = _median(lambda: O.batch_decode_attention(Q, K, V, p, scale, calib_o, "async"), args.reps)
        r["port_over_reference"] = r["port_s"] / r["reference_s"]
        print(json.dumps(r), flush=True)
        i += 1
    for n, k, m, a_, b in gem:
        row = out["ops"][i]
        for name, fo in (("ImplA", lambda: O.impl_a_gemv(a_, b)), ("ImplB", lambda: O.impl_b_flat(a_, b, cores)),
                         ("ImplC", lambda: O.impl_c_blocked(a_, b))):
            row[f"{name}_port_s"] = _median(fo, args.reps)
        row["port_over_reference_ImplA"] = row["ImplA_port_s"] / row["ImplA_reference_s"]
        print(json.dumps(row), flush=True)
        i += 1
    dst = os.path.join(ROOT, "profiles", "r2", "cpu_port_calibration.json")
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    json.dump(out, open(dst, "w"), indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main()
