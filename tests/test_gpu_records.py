"""The reference's record surface on the device kernels (records.py; reference
cli.py:98-205, record format pipeline.py:166-197): every record parses with
parse_record and carries the reference's keys."""

import pytest

pytestmark = pytest.mark.gpu

REF_KEYS = {
    "bench-gemm": {"record", "backend", "m", "n", "k", "b_n", "double_buffer", "parallelism", "median_s", "mad_s",
                   "gflops", "max_err", "status"},
    "bench-gemm-best": {"record", "backend", "n", "k", "best_b_n", "double_buffer", "parallelism_ok"},
    "bench-attn": {"record", "backend", "mode", "m", "seq", "head_dim", "p", "median_s", "mad_s", "rescale_ops",
                   "rows_recomputed"},
    "bench-attn-summary": {"record", "backend", "async_faster", "note"},
    "decode-gemm": {"record", "op", "impl", "max_err"},
    "decode-layer": {"record", "model", "batch", "seq", "mode", "max_err", "rows_recomputed", "rescale_ops",
                     "status"},
}


def test_records_parse_with_reference_keys():
    from paper_2311_01282_b200 import records
    from paper_2311_01282_b200.pipeline import format_record, parse_record
    lines = []

    def emit(f):
        lines.append(format_record(f))

    records.bench_gemm([(1024, 512)], m=8, reps=3, seed=0, emit=emit)
    records.bench_attn(seq=256, reps=3, seed=0, emit=emit)
    records.bench_prefill(seq=512, reps=3, seed=0, emit=emit, rows=(16, 64), kv_heads=2)
    assert records.decode_records("llama2-7b", batch=2, seq=64, mode="async", seed=0, reps=0, emit=emit, scale=8)
    seen = set()
    for ln in lines:
        rec = parse_record(ln)
        kind = rec["record"]
        seen.add(kind)
        if kind in REF_KEYS:
            assert REF_KEYS[kind] <= set(rec), (kind, REF_KEYS[kind] - set(rec))
        if kind in ("bench-gemm", "bench-attn-prefill", "decode-layer"):
            assert rec["status"] == "PASS", ln
    assert seen >= set(REF_KEYS) | {"bench-attn-prefill"}
