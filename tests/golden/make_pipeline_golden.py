"""Golden fixtures for the one-layer decode step, from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \\
        python tests/golden/make_pipeline_golden.py

Runs ``flatdecode.pipeline.decode_layer`` (pipeline.py:88-149) on scaled
presets and writes pipeline.npz: per case the layer output, the reference's
f64 layer oracle, its max_err, the dispatch choices and the AttnStats.  The
inputs are not stored: both sides regenerate them from ``default_rng(seed)``
(pipeline.py:94-99), which tests/test_host_logic.py pins on the CPU by
comparing the first draws.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import flatdecode as fd  # noqa: E402
fdp = sys.modules.get("flatdecode.pipeline") or __import__("flatdecode.pipeline", fromlist=["x"])

OUT = os.path.dirname(os.path.abspath(__file__))
CALIB = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=0.999989)

# (preset, scale, batch, seq_len, mode, split, seed, (m1, m2))
CASES = [
    ("llama2-7b", 16, 4, 64, "async", None, 0, (8, 64)),
    ("llama2-7b", 16, 1, 300, "sync", 3, 1, (8, 64)),
    ("chatglm2-6b-shape", 16, 16, 128, "async", 4, 2, (8, 64)),
    ("llama2-7b", 8, 9, 96, "reference", None, 3, (2, 8)),
]


def main():
    out = {}
    for i, (name, scale, batch, L, mode, split, seed, (m1, m2)) in enumerate(CASES):
        cfg = fdp.get_preset(name, scale)
        t = fd.DispatchTable(fingerprint="golden")
        for n, k in cfg.gemm_shapes().values():
            t.add(fd.DispatchEntry(n=n, k=k, m1=m1, m2=m2))
        r = fdp.decode_layer(cfg, batch, L, CALIB, t, mode, seed=seed, split=split)
        out[f"c{i}_output"] = r.output
        out[f"c{i}_oracle"] = r.oracle
        out[f"c{i}_max_err"] = np.float64(r.max_err)
        out[f"c{i}_choices"] = np.array([r.choices[op].value for op in ("kqv", "o_proj", "ffn1", "ffn2")])
        st = r.attn_stats
        out[f"c{i}_stats"] = np.array([st.rows_recomputed, st.rescale_ops, st.max_ops], dtype=np.int64)
        print(name, scale, batch, L, mode, "max_err", r.max_err, "passed", r.passed)
    rng = np.random.default_rng(0)
    out["rng0_first"] = rng.standard_normal((4,), dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **out)


if __name__ == "__main__":
    main()
