"""One-layer decode step (reference pipeline.py:24-197): host-side pieces on
the CPU, and the device layer against the reference's decode_layer outputs
(tests/golden/pipeline.npz, made by tests/golden/make_pipeline_golden.py)."""

import math
import os

import numpy as np
import pytest

from paper_2311_01282_b200 import pipeline as P

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pipeline.npz")
CASES = [  # mirrors make_pipeline_golden.CASES
    ("llama2-7b", 16, 4, 64, "async", None, 0, (8, 64)),
    ("llama2-7b", 16, 1, 300, "sync", 3, 1, (8, 64)),
    ("chatglm2-6b-shape", 16, 16, 128, "async", 4, 2, (8, 64)),
    ("llama2-7b", 8, 9, 96, "reference", None, 3, (2, 8)),
]
OPS = ("kqv", "o_proj", "ffn1", "ffn2")


def _np_oracle(cfg, w, x, kc, vc, scale):
    """numpy f64 restatement of _oracle_layer (pipeline.py:152-163) -- test-side only."""
    hd = cfg.head_dim
    q = (x.astype(np.float64) @ w["kqv"].astype(np.float64))[:, :cfg.d]
    att = np.empty_like(q)
    for h in range(cfg.n_heads):
        s = scale * q[:, h * hd:(h + 1) * hd] @ kc[h].astype(np.float64).T
        e = np.exp(s - s.max(1, keepdims=True))
        att[:, h * hd:(h + 1) * hd] = (e / e.sum(1, keepdims=True)) @ vc[h].astype(np.float64)
    o = att @ w["o_proj"].astype(np.float64)
    return ((o @ w["ffn1"].astype(np.float64)) @ w["ffn2"].astype(np.float64)).astype(np.float32)


def test_layer_config_and_presets():
    c = P.get_preset("llama2-7b")
    assert c.head_dim == 128
    assert c.gemm_shapes() == {"kqv": (12288, 4096), "o_proj": (4096, 4096),
                               "ffn1": (11008, 4096), "ffn2": (4096, 11008)}
    s = P.get_preset("chatglm2-6b-shape", 16)
    assert (s.name, s.d, s.ffn_dim, s.n_heads) == ("chatglm2-6b-shape/16", 256, 856, 2)
    with pytest.raises(KeyError):
        P.get_preset("gpt2")
    with pytest.raises(ValueError):
        P.get_preset("llama2-7b", 3)
    with pytest.raises(ValueError):
        P.get_preset("llama2-7b", 0)
    with pytest.raises(ValueError):
        P.LayerConfig("x", d=100, ffn_dim=8, n_heads=3)
    with pytest.raises(ValueError):
        P.LayerConfig("x", d=0, ffn_dim=8, n_heads=1)


def test_records_round_trip():
    rec = {"model": "llama2-7b", "batch": 4, "ms": 1.25}
    line = P.format_record(rec)
    assert line == "model=llama2-7b batch=4 ms=1.25"
    assert P.parse_record(line) == {"model": "llama2-7b", "batch": "4", "ms": "1.25"}
    with pytest.raises(ValueError):
        P.format_record({"a": "x y"})
    with pytest.raises(ValueError):
        P.format_record({"a": "x=y"})
    with pytest.raises(ValueError):
        P.parse_record("a=1 junk")
    text = "# header a=1\nnot a record\na=1 b=2\n=bad c=3\n  c=4  \n"
    assert P.parse_records(text) == [{"a": "1", "b": "2"}, {"c": "4"}]


def test_seeded_inputs_match_reference_oracle():
    """Our draw order reproduces the reference's inputs: the f64 layer oracle
    on them equals the reference's stored oracle."""
    g = np.load(GOLD)
    assert np.array_equal(np.random.default_rng(0).standard_normal((4,), dtype=np.float32), g["rng0_first"])
    for i, (name, scale, batch, L, mode, split, seed, _) in enumerate(CASES):
        cfg = P.get_preset(name, scale)
        w, x, kc, vc = P._seeded_inputs(cfg, batch, L, seed)
        ora = _np_oracle(cfg, w, x, kc, vc, 1.0 / math.sqrt(cfg.head_dim))
        err = float((np.abs(ora - g[f"c{i}_oracle"]).max(1) / np.abs(g[f"c{i}_oracle"]).max(1)).max())
        assert err <= 1e-5, (i, err)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_decode_layer_matches_reference(i):
    import importlib
    from paper_2311_01282_b200.metrics import rel_error_rowwise
    D = importlib.import_module("paper_2311_01282_b200.dispatch")
    g = np.load(GOLD)
    name, scale, batch, L, mode, split, seed, (m1, m2) = CASES[i]
    cfg = P.get_preset(name, scale)
    t = D.DispatchTable(fingerprint="golden")
    for n, k in cfg.gemm_shapes().values():
        t.add(D.DispatchEntry(n=n, k=k, m1=m1, m2=m2))
    calib = P.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=0.999989)
    r = P.decode_layer(cfg, batch, L, calib, t, mode, seed=seed, split=split)
    # same decisions and counters as the reference's decode_layer
    assert [r.choices[op].value for op in OPS] == list(g[f"c{i}_choices"])
    st = r.attn_stats
    assert [st.rows_recomputed, st.rescale_ops, st.max_ops] == list(g[f"c{i}_stats"])
    # the device f64 oracle equals the reference's oracle; the fp16 layer is within the bar
    assert rel_error_rowwise(r.oracle, g[f"c{i}_oracle"]) <= 1e-5
    assert rel_error_rowwise(r.output, g[f"c{i}_output"]) <= P.LAYER_TOLERANCE
    assert r.max_err <= P.LAYER_TOLERANCE and r.passed, (r.max_err, r.gemm_errors)
