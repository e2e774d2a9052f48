"""Per-CTA phase timeline of one lone K2 launch (build with TP_NVCC_EXTRA=-DTP_GEMM_TRACE):
start, TMA after griddepcontrol.wait, first MMA, last accumulator committed, drain done,
reducer spin start / end, reduction done, CTA end — percentiles over CTAs, us from the
earliest start.

    python scripts/gemm_trace.py [--shape gu] [--n 48]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_04104_b200 import _lib  # noqa: E402

SH = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008)}
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="gu,qkv,o,down")
ap.add_argument("--n", default="1,48")
args = ap.parse_args()
lib = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
names = ["start", "tma_pdl", "mma_first", "mma_last", "drain_done", "spin_start", "spin_end", "red_done", "end"]
for shape in args.shape.split(","):
    n_out, k = SH[shape]
    w = (torch.randn(n_out, k, device="cuda") * 0.02).to(torch.bfloat16)
    for n in [int(x) for x in args.n.split(",")]:
        x = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        out = torch.empty(n, n_out, device="cuda")
        ms = C.c_float()
        _lib.check(lib.tp_debug_gemm_timed(0, w.data_ptr(), x.data_ptr(), n, n_out, k, out.data_ptr(), 5,
                                           C.byref(ms), st))
        buf.zero_()
        _lib.check(lib.tp_debug_gemm_trace(0, buf.data_ptr()))
        _lib.check(lib.tp_debug_gemm_timed(0, w.data_ptr(), x.data_ptr(), n, n_out, k, out.data_ptr(), 1,
                                           C.byref(ms), st))
        _lib.check(lib.tp_debug_gemm_trace(0, None))
        t = buf.view(148, 32)[:, :9].cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        row = []
        for i, nm in enumerate(names):
            v = rel[:, i][t[:, i] > 0]
            if v.size:
                row.append(f"{nm} {np.percentile(v, 5):5.1f}/{np.median(v):5.1f}/{v.max():5.1f}")
        print(f"{shape:5s} n={n:3d} ({ms.value * 1e3:5.1f} us): " + "  ".join(row), flush=True)
