"""K2 alone: event-timed back-to-back launches of the tcgen05 weight-streaming GEMM
at the Llama layer shapes, vs torch (cuBLAS) bf16 at the same tiny M.

    python scripts/gemm_bench.py [--model 7b] [--iters 50]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04104_b200 import _lib  # noqa: E402

SHAPES = {"7b": [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008),
                 ("head", 32000, 4096)],
          "13b": [("qkv", 15360, 5120), ("o", 5120, 5120), ("gu", 27648, 5120), ("down", 5120, 13824)],
          "70b": [("qkv", 10240, 8192), ("o", 8192, 8192), ("gu", 57344, 8192), ("down", 8192, 28672)]}

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--n", default="1,16,48,64")
ap.add_argument("--shapes", default="", help="comma list of shape names to run (default all)")
args = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.
lib = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
for name, n_out, k in SHAPES[args.model]:
    if args.shapes and name not in args.shapes.split(","):
        continue
    w = (torch.randn(n_out, k, device="cuda") * 0.02).to(torch.bfloat16)
    for n in [int(x) for x in args.n.split(",")]:
        x = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        out = torch.empty(n, n_out, device="cuda")
        ms = C.c_float()
        _lib.check(lib.tp_debug_gemm_timed(0, w.data_ptr(), x.data_ptr(), n, n_out, k, out.data_ptr(), args.iters,
                                           C.byref(ms), st))
        ref = (x.float() @ w.float().t())
        err = (out - ref).abs().max().item() / ref.abs().max().item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        y = x @ w.t()
        e0.record()
        for _ in range(args.iters):
            y = x @ w.t()
        e1.record()
        torch.cuda.synchronize()
        tms = e0.elapsed_time(e1) / args.iters
        by = n_out * k * 2 + n * k * 2
        print(f"{name:5s} n={n:3d} {n_out}x{k}: ours {ms.value * 1e3:7.1f} us {by / ms.value / 1e6:7.0f} GB/s "
              f"({by / ms.value / 1e6 / peak:5.1%})  cublas {tms * 1e3:7.1f} us {by / tms / 1e6:7.0f} GB/s  "
              f"relerr {err:.1e}", flush=True)
