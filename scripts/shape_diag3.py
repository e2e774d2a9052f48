"""K2 alone at the 7B layer shapes (tp_debug_gemm) vs float64, n = 1 and 16."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_04104_b200 import _lib

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64); d = a - b
    return float(np.abs(d).max() / np.abs(b).max()), float(np.sqrt((d * d).mean() / (b * b).mean()))

g = torch.Generator(device="cuda").manual_seed(0)
for n_out, k in [(4096, 4096), (12288, 4096), (22016, 4096), (4096, 11008), (5120, 13824), (8192, 28672)]:
    w = (torch.rand((n_out, k), device="cuda", generator=g) * 2 - 1).mul(np.sqrt(3.0 / k)).to(torch.bfloat16)
    for n in (1, 16, 64):
        x = torch.randn((n, k), device="cuda", generator=g).to(torch.bfloat16)
        out = torch.empty((n, n_out), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().tp_debug_gemm(0, w.data_ptr(), x.data_ptr(), n, n_out, k, out.data_ptr(), _lib.stream_handle()))
        want = x.double() @ w.double().t()
        print(n_out, k, n, "k2 vs f64", rel(out.cpu().numpy(), want.cpu().numpy()),
              "torch f32 vs f64", rel((x.float() @ w.float().t()).cpu().numpy(), want.cpu().numpy()))
