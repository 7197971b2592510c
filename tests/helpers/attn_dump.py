"""Helper for tests/test_gpu_attention.py::test_incluster_recompute_matches_two_launch:
run a fixed set of injected-row attention cases and save outputs / flags to
an .npz (the caller runs it with FDPP_ATTN_INCLUSTER=0 and =1)."""

import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2311_01282_b200 as fd  # noqa: E402

CASES = [  # (B, Hq, Hkv, L, injected (b, kv-head) groups)
    (2, 8, 8, 700, [(0, 1), (1, 5)]),          # MHA, CUDA cores
    (1, 32, 32, 1024, [(0, 7)]),                # configs[0] shape
    (2, 32, 2, 1500, [(1, 0)]),                 # MQA, tensor cores
    (4, 16, 2, 2048, [(0, 0), (3, 1), (2, 1)]),  # GQA G = 8
]


def main(path):
    torch.cuda.set_device(0)
    cal = fd.ScalingCalibration(phi=-7.775933742523193, a=-1.0, b=16.577659606933594, coverage=1.0)
    out = {}
    for i, (B, Hq, Hkv, L, inj) in enumerate(CASES):
        g = torch.Generator(device="cuda").manual_seed(100 + i)
        q = torch.randn((B, Hq, 128), generator=g, device="cuda").half()
        k = torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()
        v = torch.randn((B, Hkv, L, 128), generator=g, device="cuda").half()
        for b, h in inj:
            k[b, h, L // 3].mul_(40.0)
        cfg = fd.AttentionConfig.auto(1 / math.sqrt(128), cal)
        o, st = fd.decode_attention(q, k, v, cfg, "async")
        out[f"o{i}"] = o.cpu().numpy()
        out[f"f{i}"] = st.row_mask.cpu().numpy()
        out[f"n{i}"] = np.array([st.rows_recomputed, fd.attention.launches(q, k, cfg)])
    np.savez(path, **out)


if __name__ == "__main__":
    main(sys.argv[1])
