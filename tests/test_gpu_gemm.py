"""GPU parity of subsystem 2 (GEMV / swap-AB tcgen05 flat GEMM / conventional
tcgen05 GEMM) through the C ABI against the oracle and the golden vectors."""

import os

import numpy as np
import pytest

from oracle import flatdecode_oracle as O
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 2e-3
REF_TOL = 1e-4  # f32 operands (the reference's own bar)
GEM = np.load(os.path.join(GOLDEN, "gemm.npz"))
LLAMA = ((12288, 4096), (4096, 4096), (11008, 4096), (4096, 11008))


@pytest.fixture(scope="module")
def fd():
    import paper_2311_01282_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.mark.parametrize("i", range(int(GEM["n_cases"])))
def test_golden_impls(i, fd):
    pre = f"g{i}_"
    a, b, ref = GEM[pre + "a"], GEM[pre + "b"], GEM[pre + "oracle"]
    # numpy f32 operands run the f32 CUDA-core forms: the reference's own 1e-4 bar
    for name, fn in (("A", fd.impl_a_gemv), ("B", fd.impl_b_flat), ("C", fd.impl_c_blocked)):
        out = fn(a, b)
        assert out.shape == ref.shape and out.dtype == np.float32
        assert fd.rel_error_rowwise(out, ref) <= REF_TOL, name
    out = fd.flat_gemm(a, b, fd.TileConfig(16, 32, double_buffer=True))
    assert fd.rel_error_rowwise(out, GEM[pre + "flat_16_32_db"]) <= REF_TOL


@pytest.mark.parametrize("M", [1, 3, 8, 13, 64, 100])
def test_f32_reference_precision(fd, torch, M):
    """float32 calls keep the reference's f32 contract (<= 1e-4 vs the f64
    oracle, test_flatgemm / test_dispatch), any M for every impl, and the
    double buffer never changes bits (flatgemm.py:219-221)."""
    N, K = 1000, 1032
    g = torch.Generator(device="cuda").manual_seed(M)
    a = torch.randn((M, K), generator=g, device="cuda")
    b = torch.randn((K, N), generator=g, device="cuda") / K ** 0.5
    ref = _oracle(a, b)
    outs = {}
    for name, fn in (("A", fd.impl_a_gemv), ("B", fd.impl_b_flat), ("C", fd.impl_c_blocked)):
        out = fn(a, b)
        assert out.dtype == torch.float32
        outs[name] = out.cpu().numpy()
        assert fd.rel_error_rowwise(outs[name], ref) <= REF_TOL, name
    db = fd.flat_gemm(a.cpu().numpy(), b.cpu().numpy(), fd.TileConfig(16, 32, double_buffer=True))
    sb = fd.flat_gemm(a.cpu().numpy(), b.cpu().numpy(), fd.TileConfig(16, 32, double_buffer=False))
    assert np.array_equal(db, sb)


def _operands(torch, M, N, K, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((M, K), generator=g, device="cuda").to(dtype)
    b = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).to(dtype)
    return a, b


def _oracle(a, b):
    return O.gemm_oracle(a.float().cpu().numpy(), b.float().cpu().numpy())


@pytest.mark.parametrize("N,K", LLAMA)
@pytest.mark.parametrize("M", [1, 2, 4, 8, 16, 32, 64])
def test_llama_shapes_all_impls(fd, torch, N, K, M):
    a, b = _operands(torch, M, N, K, M + N, torch.float16)
    pw = fd.pack_weight(b)
    ref = _oracle(a, b)
    from paper_2311_01282_b200 import dispatch as _  # noqa: F401
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    choices = [D.KernelChoice.IMPL_B, D.KernelChoice.IMPL_C]
    if M <= 8:
        choices.append(D.KernelChoice.IMPL_A)
    errs = {}
    for ch in choices:
        out = D.run_device(ch, a, pw)
        errs[ch.value] = fd.rel_error_rowwise(out.float().cpu().numpy(), ref)
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("N,K,M", [(12288, 4096, 128), (4096, 4096, 256), (4096, 11008, 96),
                                   (11008, 4096, 200), (22016, 4096, 256)])
def test_conventional_regime(fd, torch, N, K, M):
    """M beyond the flat band (the reference's sweep reaches 256, dispatch.py:24):
    ImplB (token tiles of 64) and ImplC (tokens on the MMA M axis; cluster
    split-K while its tiles fit one wave, stream-K beyond) against the oracle."""
    a, b = _operands(torch, M, N, K, 7 * M + N, torch.float16)
    pw = fd.pack_weight(b)
    ref = _oracle(a, b)
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    errs = {}
    for ch in (D.KernelChoice.IMPL_B, D.KernelChoice.IMPL_C):
        out = D.run_device(ch, a, pw)
        errs[ch.value] = fd.rel_error_rowwise(out.float().cpu().numpy(), ref)
        assert torch.equal(out, D.run_device(ch, a, pw))   # bitwise rerun
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("N,K,M,dt", [(12288, 4096, 256, "float16"), (1408 + 11 * 1024, 1024, 129, "float16"),
                                      (22016, 4096, 192, "float16"), (12288, 4096, 200, "bfloat16")])
def test_conventional_cta_pair(fd, torch, N, K, M, dt):
    """ImplC beyond 128 tokens on 2-CTA clusters (tcgen05.mma.cta_group::2):
    against the oracle, with a residual, a partial last pair (N % 256 != 0),
    the two-pairs-per-SM-pair ring ([22016, 4096]) and bf16; the plan query
    confirms the pair path is the one that ran; bitwise reruns."""
    from paper_2311_01282_b200 import gemm
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    dtype = getattr(torch, dt)
    a, b = _operands(torch, M, N, K, 3 * M + N, dtype)
    pw = fd.pack_weight(b)
    assert gemm.plan(2, M, N, K)[1:] == (2, 256)
    r = (torch.randn((M, N), device="cuda") * 0.1).to(dtype)
    out = D.run_device(D.KernelChoice.IMPL_C, a, pw, residual=r)
    ref = _oracle(a, b) + r.float().cpu().numpy()
    tol = TOL if dt == "float16" else 8e-3
    assert fd.rel_error_rowwise(out.float().cpu().numpy(), ref) <= tol
    assert torch.equal(out, D.run_device(D.KernelChoice.IMPL_C, a, pw, residual=r))


def test_bf16(fd, torch):
    a, b = _operands(torch, 16, 4096, 4096, 5, torch.bfloat16)
    ref = _oracle(a, b)
    for fn in (fd.impl_b_flat, fd.impl_c_blocked):
        assert fd.rel_error_rowwise(fn(a, b).float().cpu().numpy(), ref) <= 8e-3  # bf16 output rounding
    assert fd.rel_error_rowwise(fd.impl_a_gemv(a[:4], b).float().cpu().numpy(), ref[:4]) <= 8e-3


def test_ring_depth_is_bit_identical(fd, torch):
    # flatgemm.py:219-221: the staging schedule never changes the arithmetic
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    a, b = _operands(torch, 24, 4096, 4096, 7, torch.float16)
    pw = fd.pack_weight(b)
    for ctas in (0, 7, 50, -3, -8):   # stream-K fixup (>0) and cluster split-K (<0) paths
        base = D.run_device(D.KernelChoice.IMPL_B, a, pw, stages=1, ctas=ctas)
        for st in (2, 4, 0):
            assert torch.equal(base, D.run_device(D.KernelChoice.IMPL_B, a, pw, stages=st, ctas=ctas))
    # rerun determinism (stream-K fixup in fixed segment order)
    for ctas in (1, 3, 148, 300, -1, -2, -5, -8):
        x = D.run_device(D.KernelChoice.IMPL_B, a, pw, ctas=ctas)
        y = D.run_device(D.KernelChoice.IMPL_B, a, pw, ctas=ctas)
        assert torch.equal(x, y)
        assert fd.rel_error_rowwise(x.float().cpu().numpy(), _oracle(a, b)) <= TOL


def test_padding_transparency(fd, torch):
    # test_flatgemm.py:117-125: gemm(M=3) == gemm(pad8)[:3] bitwise, pad rows zero
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    a, b = _operands(torch, 3, 640, 512, 9, torch.float16)
    pw = fd.pack_weight(b)
    direct = D.run_device(D.KernelChoice.IMPL_B, a, pw, block_x=16)
    padded = D.run_device(D.KernelChoice.IMPL_B, fd.pad_rows(a, 8), pw, block_x=16)
    assert torch.equal(direct, padded[:3])
    assert not padded[3:].any()


def test_residual_epilogue(fd, torch):
    D = __import__("importlib").import_module("paper_2311_01282_b200.dispatch")
    a, b = _operands(torch, 8, 4096, 4096, 11, torch.float16)
    pw = fd.pack_weight(b)
    r = torch.randn((8, 4096), device="cuda").half()
    for ch in (D.KernelChoice.IMPL_A, D.KernelChoice.IMPL_B, D.KernelChoice.IMPL_C):
        out = D.run_device(ch, a, pw, residual=r)
        ref = _oracle(a, b) + r.float().cpu().numpy()
        assert fd.rel_error_rowwise(out.float().cpu().numpy(), ref) <= TOL


def test_ragged_and_errors(fd):
    rng = np.random.default_rng(6)
    a = rng.standard_normal((7, 101), dtype=np.float32)
    b = rng.standard_normal((101, 53), dtype=np.float32)
    ref = O.gemm_oracle(a, b)   # numpy f32: the f32 path, K = 101 zero-padded to 104
    for fn in (fd.impl_a_gemv, fd.impl_b_flat, fd.impl_c_blocked):
        assert fd.rel_error_rowwise(fn(a, b), ref) <= REF_TOL
    with pytest.raises(fd.ShapeError):
        fd.impl_a_gemv(np.ones((1, 2), np.float32), np.ones((3, 4), np.float32))
    eye = np.eye(64, dtype=np.float32)
    x = np.random.default_rng(3).standard_normal((64, 64)).astype(np.float16).astype(np.float32)
    assert np.array_equal(fd.impl_c_blocked(x, eye), x)        # identity exact through fp16


def test_profile_shape_real(fd, torch):
    details = []
    e = fd.profile_shape(4096, 4096, m_sweep=(1, 2, 4, 8, 16, 32, 64), reps=5, details=details)
    assert 1 <= e.m1 <= e.m2
    sweep = [d["m"] for d in details]
    m1, m2 = O.decide(sweep, [d["ImplA"] for d in details], [d["ImplB"] for d in details],
                      [d["ImplC"] for d in details])
    assert (e.m1, e.m2) == (m1, m2)      # native decision == oracle decision on the same medians
