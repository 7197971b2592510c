"""GPU parity of subsystem 1 (async-softmax split-KV attention) through the
C ABI against the reference's golden vectors and the oracle.

Bars (north_star): outputs within 2e-3 relative (rowwise, metrics.py:19-32),
recompute-flag sets bit-exact, AttnStats arithmetic exact, reruns bitwise."""

import math
import os

import numpy as np
import pytest

from oracle import flatdecode_oracle as O
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 2e-3          # north_star bar for fp16/bf16 storage
TOL_F32 = 2e-5      # fp32 inputs: only summation order differs from the oracle
TOL_BF16 = 4e-3     # bf16 OUTPUT rounding alone is up to 2^-8 = 3.9e-3 of the row max

ATT = np.load(os.path.join(GOLDEN, "attention.npz"))


@pytest.fixture(scope="module")
def fd():
    import paper_2311_01282_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _case(i, fd):
    pre = f"c{i}_"
    meta = ATT[pre + "meta"]
    calib = fd.ScalingCalibration(phi=float(meta[2]), a=float(meta[3]), b=float(meta[4]),
                                  coverage=1.0)
    cfg = fd.AttentionConfig(p=int(meta[0]), scale=float(meta[1]), calib=calib)
    return ATT[pre + "Q"], ATT[pre + "K"], ATT[pre + "V"], cfg, pre


@pytest.mark.parametrize("i", range(int(ATT["n_cases"])))
def test_golden_async_sync(i, fd):
    Q, K, V, cfg, pre = _case(i, fd)
    out, st = fd.batch_decode_attention(Q, K, V, cfg, "async")
    assert fd.rel_error_rowwise(out, ATT[pre + "out_async"]) <= TOL_F32
    assert np.array_equal(st.row_mask.numpy(), ATT[pre + "redo"])
    assert [st.rows_recomputed, st.rescale_ops, st.max_ops] == ATT[pre + "stats_async"].tolist()
    out, st = fd.batch_decode_attention(Q, K, V, cfg, "sync")
    assert fd.rel_error_rowwise(out, ATT[pre + "out_sync"]) <= TOL_F32
    assert [st.rows_recomputed, st.rescale_ops, st.max_ops] == ATT[pre + "stats_sync"].tolist()
    out, _ = fd.batch_decode_attention(Q, K, V, cfg, "reference")
    assert fd.rel_error_rowwise(out, ATT[pre + "out_ref"]) <= 1e-6


@pytest.mark.parametrize("i", range(int(ATT["n_cases"])))
def test_golden_chunk_states(i, fd):
    Q, K, V, cfg, pre = _case(i, fd)
    num, den, viol = fd.async_partials(Q, K, V, cfg)
    assert np.array_equal(viol, ATT[pre + "viol"])          # first violating key, bit-exact
    gden = ATT[pre + "den"].astype(np.float32)
    ok = np.isfinite(gden)
    assert np.allclose(den[ok], gden[ok], rtol=1e-5, atol=1e-30)
    gnum = ATT[pre + "num"].astype(np.float32)
    M, p, d = gnum.shape
    fin = np.isfinite(gnum).all(axis=2).reshape(-1)
    if fin.any():
        a = num.reshape(M * p, d)[fin]
        g = gnum.reshape(M * p, d)[fin]
        if np.abs(g).max() > 0:
            assert fd.rel_error_rowwise(a, g) <= 1e-5


def test_worked_example_state(fd):
    # test_attention.py:95-143: phi=6, band (-3, 3), K = I
    calib = fd.ScalingCalibration(phi=6.0, a=-3.0, b=3.0, coverage=1.0)
    cfg = fd.AttentionConfig(p=2, scale=1.0, calib=calib)
    K = np.eye(4, dtype=np.float32)
    V = np.random.default_rng(7).standard_normal((4, 4)).astype(np.float32)
    q = np.array([4.0, 5.0, 9.5, 7.0], np.float32)
    st = fd.async_chunk_state(q, K, V, 2, 4, cfg)
    assert st.overflow_index == 2 and st.den == 0.0 and not st.num.any()
    o, rec = fd.decode_attention_async(q, K, V, cfg)
    assert rec
    assert np.array_equal(o, fd.decode_attention_sync(q, K, V, cfg))


def _qkv(torch, B, Hq, Hkv, L, D, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((B, Hq, D), generator=g, device="cuda").to(dtype)
    k = torch.randn((B, Hkv, L, D), generator=g, device="cuda").to(dtype)
    v = torch.randn((B, Hkv, L, D), generator=g, device="cuda").to(dtype)
    return q, k, v


def _oracle_batched(q, k, v, p, scale, calib):
    """Run the oracle per (b, kv-head) with the G query rows of that group."""
    B, Hq, D = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    qn, kn, vn = (t.float().cpu().numpy() for t in (q, k, v))
    out = np.zeros((B, Hq, D), np.float32)
    redo = np.zeros((B, Hq), bool)
    clear = np.ones((B, Hq), bool)
    for b in range(B):
        for h in range(Hkv):
            Qg = qn[b, h * G:(h + 1) * G]
            o, _, r = O.batch_decode_attention(Qg, kn[b, h], vn[b, h], p, scale, calib, "async")
            out[b, h * G:(h + 1) * G] = o
            redo[b, h * G:(h + 1) * G] = r
            c, _ = O.row_guard_ok(Qg, kn[b, h], scale, calib)
            clear[b, h * G:(h + 1) * G] = c
    return out, redo, clear


GOLD_CAL = (-7.775933742523193, -1.0, 16.577659606933594)


@pytest.mark.parametrize("dtype_name", ["float16", "bfloat16"])
def test_config1_llama_mha(fd, torch, dtype_name):
    # config 1: batch 1, 32 heads x 128, L=1024, N(0,1) inputs, golden calibration
    dtype = getattr(torch, dtype_name)
    q, k, v = _qkv(torch, 1, 32, 32, 1024, 128, 0, dtype)
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    cfg = fd.AttentionConfig(p=4, scale=1 / math.sqrt(128), calib=calib)
    o, st = fd.decode_attention(q, k, v, cfg, "async")
    oc = O.Calib(*GOLD_CAL)
    ref, redo, clear = _oracle_batched(q, k, v, 4, cfg.scale, oc)
    assert clear.all()
    assert st.rows_recomputed == 0 and not redo.any()
    tol = TOL if dtype == torch.float16 else TOL_BF16
    assert fd.rel_error_rowwise(o.float().cpu().numpy().reshape(-1, 128), ref.reshape(-1, 128)) <= tol
    o2, _ = fd.decode_attention(q, k, v, cfg, "async")
    assert torch.equal(o, o2)                                   # bitwise rerun


def test_mqa_recompute_flags(fd, torch):
    # config 4 shape family (MQA, G=16) at reduced L: inject rows x12 outside the band
    B, Hq, Hkv, L, D = 2, 32, 2, 2048, 128
    q, k, v = _qkv(torch, B, Hq, Hkv, L, D, 1, torch.float16)
    inject = [(0, 3), (0, 17), (1, 30), (1, 0), (1, 5)]
    for b, h in inject:
        q[b, h] = (q[b, h].float() * 12).half()
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    for p, spc in ((4, 0), (7, 3), (1, 1)):
        cfg = fd.AttentionConfig(p=p, scale=1 / math.sqrt(D), calib=calib, splits_per_chunk=spc)
        o, st = fd.decode_attention(q, k, v, cfg, "async")
        ref, redo, clear = _oracle_batched(q, k, v, p, cfg.scale, O.Calib(*GOLD_CAL))
        assert clear.all()
        assert np.array_equal(st.row_mask.cpu().numpy(), redo)   # flag set bit-exact
        assert st.rows_recomputed == len(inject)
        assert st.rescale_ops == 2 * len(inject) * p
        assert st.max_ops == len(inject) * (p + 1)
        assert fd.rel_error_rowwise(o.float().cpu().numpy().reshape(-1, D), ref.reshape(-1, D)) <= TOL


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16])
def test_gqa_groups_sync_and_async(fd, torch, G):
    Hkv = 2
    q, k, v = _qkv(torch, 2, Hkv * G, Hkv, 777, 128, 3 + G, torch.float16)
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    cfg = fd.AttentionConfig(p=3, scale=1 / math.sqrt(128), calib=calib)
    ref, _, _ = _oracle_batched(q, k, v, 3, cfg.scale, O.Calib(*GOLD_CAL))
    for mode in ("async", "sync"):
        o, _ = fd.decode_attention(q, k, v, cfg, mode)
        assert fd.rel_error_rowwise(o.float().cpu().numpy().reshape(-1, 128), ref.reshape(-1, 128)) <= TOL


@pytest.mark.parametrize("inject", [0, 1, 5])
def test_acceptance_criterion_3(fd, inject):
    # test_acceptance.py:92-112 through the drop-in API: r rows recomputed, exact count
    rng = np.random.default_rng(33 + inject)
    calib = fd.ScalingCalibration(phi=0.0, a=-8.0, b=8.0, coverage=1.0)
    worst = 0.0
    for _ in range(25):
        M, L, d = 8, 64, 16
        K = rng.standard_normal((L, d), dtype=np.float32)
        V = rng.standard_normal((L, d), dtype=np.float32)
        Q = rng.standard_normal((M, d), dtype=np.float32)
        lg = Q.astype(np.float64) @ K.astype(np.float64).T
        Q *= (6.0 / np.abs(lg).max(axis=1, keepdims=True)).astype(np.float32)
        rows = rng.choice(M, size=inject, replace=False)
        Q[rows] *= 3.0
        cfg = fd.AttentionConfig(p=4, scale=1.0, calib=calib)
        out, st = fd.batch_decode_attention(Q, K, V, cfg, "async")
        assert st.rows_recomputed == inject
        worst = max(worst, fd.rel_error_rowwise(out, O.attention_reference(Q, K, V, 1.0)))
    assert worst <= 1e-5


def test_adversarial_span_sync(fd):
    d = 8
    K = np.eye(d, dtype=np.float32)
    V = np.random.default_rng(5).standard_normal((d, d)).astype(np.float32)
    q = np.array([40.0, -40.0, 20.0, -20.0, 0.0, 10.0, -10.0, 30.0], dtype=np.float32)
    out = fd.decode_attention_sync(q, K, V, fd.AttentionConfig(p=4, scale=1.0))
    assert fd.rel_error_rowwise(out, O.attention_reference(q[None], K, V, 1.0)[0]) <= 1e-5


def test_errors(fd):
    Q = np.ones((1, 8), np.float32)
    with pytest.raises(ValueError):
        fd.batch_decode_attention(Q, np.ones((4, 8), np.float32), np.ones((4, 8), np.float32),
                                  fd.AttentionConfig(p=2, scale=1.0), "turbo")
    with pytest.raises(ValueError, match="alibration"):
        fd.batch_decode_attention(Q, np.ones((4, 8), np.float32), np.ones((4, 8), np.float32),
                                  fd.AttentionConfig(p=2, scale=1.0), "async")
    with pytest.raises(fd.ShapeError):
        fd.batch_decode_attention(np.ones((2, 3), np.float32), np.ones((4, 5), np.float32),
                                  np.ones((4, 5), np.float32), fd.AttentionConfig(p=1, scale=1.0), "sync")
    with pytest.raises(ValueError):
        fd.batch_decode_attention(Q, np.ones((4, 8), np.float32), np.ones((4, 8), np.float32),
                                  fd.AttentionConfig(p=9, scale=1.0), "sync")


def test_sample_logits_and_calibrate(fd, torch):
    """Calibration producer: device-sampled logits equal scale * q . k at the
    returned indices; calibrate() on them covers the sample (softmax.py:219-266)."""
    B, Hq, Hkv, L, D = 3, 8, 2, 300, 128
    q, k, _ = _qkv(torch, B, Hq, Hkv, L, D, 11, torch.float16)
    lens = torch.tensor([300, 17, 123], dtype=torch.int32, device="cuda")
    s, idx = fd.sample_logits(q, k, 0.125, 4096, seq_lens=lens, seed=3, return_index=True)
    idx = idx.long().cpu()
    assert (idx[:, 2] < lens.cpu()[idx[:, 0]].long()).all()
    G = Hq // Hkv
    ref = 0.125 * (q.float()[idx[:, 0], idx[:, 1]] * k.float()[idx[:, 0], idx[:, 1] // G, idx[:, 2]]).sum(-1)
    assert torch.allclose(s.cpu(), ref.cpu(), rtol=1e-5, atol=1e-5)
    cal = fd.calibrate(s.cpu().numpy(), 0.9999, 1.0)
    x = s.cpu().numpy() - cal.phi
    assert ((x > cal.a) & (x < cal.b)).mean() >= 0.9999


def test_vector_softmax_apis_match_golden(fd):
    """softmax_reference / softmax_unified / partial_softmax_sync (SURVEY §8a rows
    a5/a6) on the device against the real reference's golden vectors."""
    import os
    S = np.load(os.path.join(os.path.dirname(__file__), "golden", "softmax.npz"))
    for i in range(int(S["n_cases"])):
        x = S[f"s{i}_x"]
        assert fd.rel_error_elementwise(fd.softmax_reference(x), S[f"s{i}_ref"]) <= 2e-6
        assert fd.rel_error_elementwise(fd.softmax_unified(x, 0.0), S[f"s{i}_unified_phi0"]) <= 2e-6
        assert fd.rel_error_elementwise(fd.softmax_unified(x, 6.0), S[f"s{i}_unified_phi6"]) <= 2e-6
        for p in (1, 2, 4):
            if p <= x.size:
                assert fd.rel_error_elementwise(fd.partial_softmax_sync(x, p), S[f"s{i}_sync_p{p}"]) <= 2e-5
        ref64 = fd.softmax_reference_f64(x.astype(np.float64))
        assert ref64.dtype == np.float64 and abs(ref64.sum() - 1.0) < 1e-12
    a = fd.softmax_unified(np.zeros(5, np.float32), 0.0)
    assert np.allclose(a, 0.2)
    with pytest.raises(fd.SoftmaxOverflow) as e:
        fd.softmax_unified(np.array([0.0, 100.0, 1.0], np.float32), 0.0)   # e^100 overflows f32
    assert e.value.index == 1
    with pytest.raises(fd.DegenerateSumError):
        fd.softmax_unified(np.array([-200.0, -300.0], np.float32), 0.0)    # all underflow
    with pytest.raises(ValueError):
        fd.softmax_unified(np.array([np.nan], np.float32), 0.0)
    with pytest.raises(ValueError):
        fd.partial_softmax_sync(np.ones(3, np.float32), 4)                  # p > n


@pytest.mark.parametrize("Hkv", [8, 1])  # MHA (CUDA cores) and G = 8 (tensor cores)
@pytest.mark.parametrize("p", [0, 3])
def test_ragged_seq_lens(fd, torch, Hkv, p):
    """Per-row attended lengths on the device (the decode step's seq_lens):
    ragged rows, a 1-key row, rows shorter than the chunk count."""
    B, Hq, L, D = 4, 8, 300, 128
    q, k, v = _qkv(torch, B, Hq, Hkv, L, D, 21 + Hkv, torch.float16)
    lens = torch.tensor([300, 1, 77, 129], dtype=torch.int32, device="cuda")
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    cfg = fd.AttentionConfig(p=p or fd.AUTO, scale=1 / math.sqrt(D), calib=calib)
    o, st = fd.decode_attention(q, k, v, cfg, "async", seq_lens=lens)
    G = Hq // Hkv
    qn, kn, vn = (t.float().cpu().numpy() for t in (q, k, v))
    for b, n in enumerate(lens.tolist()):
        for h in range(Hq):
            ref = O.attention_reference(qn[b, h][None], kn[b, h // G, :n], vn[b, h // G, :n], cfg.scale)
            assert fd.rel_error_rowwise(o[b, h][None].float().cpu().numpy(), ref) <= TOL
    assert st.rows_recomputed == 0


def test_incluster_recompute_matches_two_launch(tmp_path):
    """The decode plans recompute flagged rows inside the async launch's cluster
    (one launch).  FDPP_ATTN_INCLUSTER=0 restores the separate list-walking
    recompute launch; FDPP_ATTN_ABORT=0 keeps streaming after a violation.
    * in-cluster, no early stop: the same arithmetic in the same order as the
      two-launch form -- outputs, flag sets and counters bitwise equal;
    * in-cluster with the early stop (default): a group that saw a violation
      stops its async stream and is recomputed whole, its flags re-derived
      from the sync pass's band check -- flag sets and counters still equal
      bitwise, outputs within the fp16 bar (its unflagged rows now come from
      the sync softmax) and bitwise on every group without a flagged row."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode, env_over in (("two", {"FDPP_ATTN_INCLUSTER": "0"}),
                           ("one", {"FDPP_ATTN_INCLUSTER": "1", "FDPP_ATTN_ABORT": "0"}),
                           # =2 forces the early stop on these short rows (auto: >= 1K keys per CTA)
                           ("abort", {"FDPP_ATTN_INCLUSTER": "1", "FDPP_ATTN_ABORT": "2"})):
        path = str(tmp_path / f"inc_{mode}.npz")
        env = dict(os.environ, **env_over)
        subprocess.run([sys.executable, os.path.join(root, "tests", "helpers", "attn_dump.py"), path],
                       check=True, env=env, cwd=root, timeout=600)
        res[mode] = np.load(path)
    two, one, ab = res["two"], res["one"], res["abort"]
    for key in two.files:
        if key.startswith("n"):
            assert two[key][0] == one[key][0] == ab[key][0] and two[key][0] > 0, key   # rows recomputed
            assert (two[key][1], one[key][1], ab[key][1]) == (2, 1, 1), key           # launches per call
        elif key.startswith("f"):
            assert np.array_equal(two[key], one[key]) and np.array_equal(two[key], ab[key]), key
        else:
            assert np.array_equal(two[key], one[key]), key
            o2, oa = two[key].astype(np.float32), ab[key].astype(np.float32)
            D = o2.shape[-1]
            assert fd_rel(oa.reshape(-1, D), o2.reshape(-1, D)) <= TOL, key
            # bitwise on the (b, kv-head) groups without a flagged row
            flags = two["f" + key[1:]]
            B, Hq = flags.shape
            i = int(key[1:])
            Hkv = __import__("tests.helpers.attn_dump", fromlist=["CASES"]).CASES[i][2]
            G = Hq // Hkv
            clean = ~flags.reshape(B, Hkv, G).any(-1)
            assert np.array_equal(o2.reshape(B, Hkv, G, D)[clean], oa.reshape(B, Hkv, G, D)[clean]), key


def fd_rel(a, b):
    return float((np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1e-8)).max())


@pytest.mark.parametrize("B,Hq,Hkv,L", [(1, 32, 32, 1024), (2, 32, 2, 1500)])
def test_incluster_recompute_vs_oracle(fd, torch, B, Hq, Hkv, L):
    # the single-launch recompute (auto plan, cluster join) against the oracle,
    # with one key far outside the band in two (b, kv-head) groups
    q, k, v = _qkv(torch, B, Hq, Hkv, L, 128, 17, torch.float16)
    groups = [(0, 0), (B - 1, Hkv - 1)]
    for b, h in groups:
        k[b, h, L // 2].mul_(40.0)
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    cfg = fd.AttentionConfig.auto(1 / math.sqrt(128), calib)
    assert fd.attention.launches(q, k, cfg) == 1
    p, _ = fd.attention.plan(q, k, cfg)
    o, st = fd.decode_attention(q, k, v, cfg, "async")
    ref, redo, clear = _oracle_batched(q, k, v, p, cfg.scale, O.Calib(*GOLD_CAL))
    assert clear.all()
    assert np.array_equal(st.row_mask.cpu().numpy(), redo)
    G = Hq // Hkv
    assert st.rows_recomputed == int(redo.sum())
    assert any(redo[b, h * G:(h + 1) * G].any() for b, h in groups)
    assert fd.rel_error_rowwise(o.float().cpu().numpy().reshape(-1, 128), ref.reshape(-1, 128)) <= TOL


def test_early_stop_ragged_lengths_vs_oracle(fd, torch):
    """The tensor-core path's early stop (auto plan, >= 1K keys per CTA) with
    ragged per-row lengths and out-of-band keys inside some rows' attended
    range (and one past a row's length, which must not flag it): flag sets
    bit-exact against the oracle's redo on each row's own prefix, outputs
    within the fp16 bar."""
    B, Hq, Hkv, L, D = 4, 32, 2, 16384, 128
    G = Hq // Hkv
    q, k, v = _qkv(torch, B, Hq, Hkv, L, D, 41, torch.float16)
    lens = torch.tensor([16384, 9000, 12001, 15999], dtype=torch.int32, device="cuda")
    k[0, 1, 5000].mul_(40.0)      # inside row 0's range
    k[1, 0, 8999].mul_(40.0)      # the last attended key of row 1
    k[2, 1, 12500].mul_(40.0)     # past row 2's length: must not flag
    calib = fd.ScalingCalibration(*GOLD_CAL, coverage=1.0)
    cfg = fd.AttentionConfig.auto(1 / math.sqrt(D), calib)
    p, _ = fd.attention.plan(q, k, cfg)
    o, st = fd.decode_attention(q, k, v, cfg, "async", seq_lens=lens)
    qn = q.float().cpu().numpy()
    flags = st.row_mask.cpu().numpy()
    oc = O.Calib(*GOLD_CAL)
    n_redo = 0
    for b, n in enumerate(lens.tolist()):
        kb = k[b, :, :n].float().cpu().numpy()
        vb = v[b, :, :n].float().cpu().numpy()
        for h in range(Hkv):
            Qg = qn[b, h * G:(h + 1) * G]
            ref, _, redo = O.batch_decode_attention(Qg, kb[h], vb[h], p, cfg.scale, oc, "async")
            clear, _ = O.row_guard_ok(Qg, kb[h], cfg.scale, oc)
            assert clear.all()
            assert np.array_equal(flags[b, h * G:(h + 1) * G], redo), (b, h)
            assert fd.rel_error_rowwise(o[b, h * G:(h + 1) * G].float().cpu().numpy(), ref) <= TOL, (b, h)
            n_redo += int(redo.sum())
    # the injected groups are flagged; row 2's key past its length is covered by the
    # bit-exact comparison with the oracle on the row's own prefix
    assert flags[0, G:2 * G].any() and flags[1, :G].any()
    assert st.rows_recomputed == n_redo
