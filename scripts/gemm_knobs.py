"""K2 alone under diagnostic knobs (tp_debug_gemm_knob): fix-up mode (0 normal,
1 skip reduction, 2 also skip partial publish, 3 reduce without waiting — WRONG
results for 1-3) and ring depth, at several node counts.

    python scripts/gemm_knobs.py [--shape gu] [--n 1,8,16,48]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04104_b200 import _lib  # noqa: E402

SH = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "head": (32000, 4096)}
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="gu")
ap.add_argument("--n", default="1,8,16,48")
ap.add_argument("--fixup", default="0,1,2")
ap.add_argument("--stages", default="8")
ap.add_argument("--iters", type=int, default=50)
args = ap.parse_args()
lib = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
for shape in args.shape.split(","):
    n_out, k = SH[shape]
    w = (torch.randn(n_out, k, device="cuda") * 0.02).to(torch.bfloat16)
    for n in [int(x) for x in args.n.split(",")]:
        x = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        out = torch.empty(n, n_out, device="cuda")
        row = []
        for stg in [int(s) for s in args.stages.split(",")]:
            for fx in [int(f) for f in args.fixup.split(",")]:
                _lib.check(lib.tp_debug_gemm_knob(0, stg))
                _lib.check(lib.tp_debug_gemm_knob(2, fx))
                ms = C.c_float()
                _lib.check(lib.tp_debug_gemm_timed(0, w.data_ptr(), x.data_ptr(), n, n_out, k, out.data_ptr(),
                                                   args.iters, C.byref(ms), st))
                row.append(f"st{stg}/fx{fx} {ms.value * 1e3:6.1f}")
        _lib.check(lib.tp_debug_gemm_knob(0, 8))
        _lib.check(lib.tp_debug_gemm_knob(2, 0))
        print(f"{shape:5s} n={n:3d}: " + "  ".join(row), flush=True)
