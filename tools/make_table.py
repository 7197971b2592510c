"""Profile every decode-step GEMM shape on this B200 with the reference's
decision flow (profile_shape: median of reps, 20%-MAD gate, _first_sustained)
and write the dispatch table plus the per-point medians."""
import importlib
import json
import sys

sys.path.insert(0, ".")
import paper_2311_01282_b200  # noqa: E402,F401
from paper_2311_01282_b200 import llama  # noqa: E402

D = importlib.import_module("paper_2311_01282_b200.dispatch")
out = sys.argv[1] if len(sys.argv) > 1 else "tables/b200_decode.tbl"
# every decode-step GEMM shape the bench can run: Llama-2-7B, ChatGLM2-6B, and
# Llama-2-70B per rank at t = 1/2/4/8, plus config 2's shapes
runs = [(llama.LLAMA2_7B, 1), (llama.CHATGLM2_6B, 1)] + [(llama.LLAMA2_70B, t) for t in (1, 2, 4, 8)]
table = D.DispatchTable(fingerprint=D.default_fingerprint())
details = {}
shapes = sorted({s for c, t in runs for s in c.gemm_shapes(t).values()} |
                {(12288, 4096), (4096, 4096), (11008, 4096), (4096, 11008)})
for n, k in shapes:
    det = []
    e = D.profile_shape(n, k, m_sweep=D.B200_M_SWEEP, reps=9, details=det)
    table.add(e)
    details[f"{n}x{k}"] = det
    print(f"[{n},{k}] m1={e.m1} m2={e.m2}  " + "  ".join(
        f"M={d['m']}:A={d['ImplA']*1e6:.1f}/B={d['ImplB']*1e6:.1f}/C={d['ImplC']*1e6:.1f}" for d in det), flush=True)
D.save_table(table, out)
json.dump(details, open(out.replace(".tbl", ".medians.json"), "w"), indent=1)
print("wrote", out)
