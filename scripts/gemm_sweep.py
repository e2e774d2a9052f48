"""K2 tuning sweep: grouped launches at the bench's per-stage node counts
(7 same-device stages, as phase 1 runs them) and the lone verify stage,
for several ring-depth / smem-budget knob settings.

    python scripts/gemm_sweep.py [--model 7b] [--iters 20]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04104_b200 import _lib  # noqa: E402

SHAPES = {"7b": [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008)]}
ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--n", default="45,35,29,23,17,11,3")
ap.add_argument("--knobs", default="8:200")
args = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(root, "MEASURED_PEAKS.json")) else 6650.0
lib = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
ns = [int(x) for x in args.n.split(",")]
for knob in args.knobs.split(","):
    parts = [int(x) for x in knob.split(":")]
    ms_, kb_ = parts[0], parts[1]
    fx = parts[2] if len(parts) > 2 else 0
    _lib.check(lib.tp_debug_gemm_knob(0, ms_))
    _lib.check(lib.tp_debug_gemm_knob(1, kb_))
    _lib.check(lib.tp_debug_gemm_knob(2, fx))
    tot_b = tot_t = 0.0
    for name, n_out, k in SHAPES[args.model]:
        for group in (ns, [1]):
            g = len(group)
            ws = [(torch.randn(n_out, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(g)]
            xs = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for n in group]
            outs = [torch.empty(n, n_out, device="cuda") for n in group]
            arr = lambda ts: (C.c_void_p * g)(*[t.data_ptr() for t in ts])  # noqa: E731
            nn = (C.c_int32 * g)(*group)
            ms = C.c_float()
            _lib.check(lib.tp_debug_gemm_group_timed(0, g, arr(ws), arr(xs), nn, n_out, k, arr(outs), args.iters,
                                                     C.byref(ms), st))
            by = g * n_out * k * 2 + sum(group) * k * 2
            gbs = by / ms.value / 1e6
            if g > 1:
                tot_b += by
                tot_t += ms.value
            print(f"fixup={fx} stages<={ms_:2d} smem={kb_}KB {name:5s} members={g} n={group}: {ms.value * 1e3:8.1f} us "
                  f"{gbs:7.0f} GB/s ({gbs / peak:6.1%})", flush=True)
            del ws, xs, outs
    print(f"stages<={ms_:2d} smem={kb_}KB grouped layer total: {tot_t * 1e3:8.1f} us "
          f"{tot_b / tot_t / 1e6:7.0f} GB/s ({tot_b / tot_t / 1e6 / peak:6.1%})", flush=True)
