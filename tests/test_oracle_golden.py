"""Pin the oracle (test infrastructure) against fixtures produced by the real
reference (tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import flatdecode_oracle as O
from tests.conftest import GOLDEN

ATT = np.load(os.path.join(GOLDEN, "attention.npz"))
GEM = np.load(os.path.join(GOLDEN, "gemm.npz"))
SMX = np.load(os.path.join(GOLDEN, "softmax.npz"))
with open(os.path.join(GOLDEN, "host.json")) as f:
    HOST = json.load(f)


def _case(i):
    pre = f"c{i}_"
    meta = ATT[pre + "meta"]
    calib = O.Calib(phi=float(meta[2]), a=float(meta[3]), b=float(meta[4]))
    return (ATT[pre + "Q"], ATT[pre + "K"], ATT[pre + "V"], int(meta[0]), float(meta[1]),
            calib, pre)


@pytest.mark.parametrize("i", range(int(ATT["n_cases"])))
def test_async_partials_match_reference(i):
    Q, K, V, p, scale, calib, pre = _case(i)
    bounds = O.chunk_bounds(K.shape[0], p)
    assert np.array_equal(bounds, ATT[pre + "bounds"])
    num, den, viol = O.async_partials(Q, K, V, scale, calib, bounds)
    # the restated numba loop is bit-identical on the violation indices
    assert np.array_equal(viol, ATT[pre + "viol"])
    ok = np.isfinite(ATT[pre + "den"])
    assert np.allclose(den[ok], ATT[pre + "den"][ok], rtol=1e-6, atol=0)
    assert np.allclose(num, ATT[pre + "num"], rtol=1e-6, atol=1e-30, equal_nan=True)


@pytest.mark.parametrize("i", range(int(ATT["n_cases"])))
def test_batch_modes_match_reference(i):
    Q, K, V, p, scale, calib, pre = _case(i)
    for mode, key in (("async", "out_async"), ("sync", "out_sync"), ("reference", "out_ref")):
        out, stats, redo = O.batch_decode_attention(Q, K, V, p, scale, calib, mode)
        assert O.rel_error_rowwise(out, ATT[pre + key]) <= 1e-6, mode
        if mode == "async":
            assert np.array_equal(redo, ATT[pre + "redo"])
            st = ATT[pre + "stats_async"]
            assert [stats["rows_recomputed"], stats["rescale_ops"], stats["max_ops"]] == st.tolist()
        if mode == "sync":
            st = ATT[pre + "stats_sync"]
            assert [stats["rows_recomputed"], stats["rescale_ops"], stats["max_ops"]] == st.tolist()


@pytest.mark.parametrize("i", range(int(GEM["n_cases"])))
def test_gemms_match_reference(i):
    pre = f"g{i}_"
    a, b = GEM[pre + "a"], GEM[pre + "b"]
    assert np.array_equal(O.gemm_oracle(a, b), GEM[pre + "oracle"])   # bit-exact f64 oracle
    assert np.array_equal(O.impl_a_gemv(a, b), GEM[pre + "implA"])
    assert np.array_equal(O.impl_b_flat(a, b, 8), GEM[pre + "implB"])
    assert np.array_equal(O.impl_c_blocked(a, b), GEM[pre + "implC"])
    assert np.array_equal(O.flat_gemm(a, b, 16, 32, double_buffer=True), GEM[pre + "flat_16_32_db"])
    assert np.array_equal(O.flat_gemm(a, b, 8, 8), GEM[pre + "flat_8_8"])


def test_softmax_unified_matches_reference():
    for i in range(int(SMX["n_cases"])):
        x = SMX[f"s{i}_x"]
        assert O.rel_error_elementwise(O.softmax_unified(x, 0.0), SMX[f"s{i}_unified_phi0"]) <= 1e-6
        assert O.rel_error_elementwise(O.softmax_unified(x, 6.0), SMX[f"s{i}_unified_phi6"]) <= 1e-6


def test_chunk_bounds():
    for n, p, exp in HOST["chunk_bounds"]:
        assert O.chunk_bounds(n, p).tolist() == exp


def test_select_tile():
    for m, n, k, w, tgt, bn, bk, mp, db in HOST["select_tile"]:
        t = O.select_tile(m, n, k, w, tgt)
        assert (t["b_n"], t["b_k"], t["m_pad"], t["double_buffer"]) == (bn, bk, mp, db)


def test_arithmetic_intensity():
    for m, n, k, bn, bk, flops, traffic, inten, par in HOST["arithmetic_intensity"]:
        f, t, i, p = O.arithmetic_intensity(m, n, k, bn, bk)
        assert (f, t, i, p) == (flops, traffic, inten, par)


def test_double_buffer_pipeline():
    for T, ev in HOST["double_buffer_pipeline"].items():
        assert [list(e) for e in O.double_buffer_pipeline(int(T))] == ev


def test_calibrate_golden():
    phi, a, b, cov = HOST["calibrate_golden"]
    c = O.calibrate(np.random.default_rng(0).normal(0.0, 2.0, 1_000_000), 0.9999, 1.0)
    assert (c.phi, c.a, c.b, c.coverage) == (phi, a, b, cov)
    for s, target, phi, a, b, cov in HOST["calibrate_small"]:
        c = O.calibrate(np.array(s), target)
        assert (c.phi, c.a, c.b, c.coverage) == (phi, a, b, cov)


def test_first_sustained_and_decisions():
    for new, old, start, exp in HOST["first_sustained"]:
        assert O.first_sustained(new, old, start) == exp
    for sweep, ma, mb, mc, m1, m2 in HOST["profile_decisions"]:
        assert O.decide(sweep, ma, mb, mc) == (m1, m2)


def test_dispatch_grid_and_table_text():
    entries = {(n, k): (m1, m2) for n, k, m1, m2 in HOST["dispatch_entries"]}
    for m, n, k, choice in HOST["dispatch_grid"]:
        assert O.dispatch(m, *entries[(n, k)]) == choice
    assert O.table_text("golden", entries) == HOST["table_text"]


def test_check_bounds_worked_example():
    c = O.Calib(phi=6.0, a=-3.0, b=3.0)
    assert O.check_bounds(np.array([4, 5, 6, 7], np.float32), c) is None
    assert O.check_bounds(np.array([4, 5, 9.5, 7], np.float32), c) == 2
    edge = O.Calib(phi=0.0, a=-1.0, b=1.0)
    assert O.check_bounds(np.array([1.0], np.float32), edge) == 0   # boundary is a violation
