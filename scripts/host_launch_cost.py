"""Host cost of one lone stage forward call (7B shape, 4 layers, n=16): full launch
sequence vs the same call with the GEMM and attention launches skipped (diagnostic
mask: WRONG results), and a bare cudaLaunchKernelEx-rate reference."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from paper_2504_04104_b200 import _lib  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel, forward_members  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner  # noqa: E402

cfg = tp.LlamaConfig.llama2_7b(layers=8)  # 7B widths, two 4-layer stages
m = LlamaModel(cfg, max_nodes=64)
prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab, 512)]
r = PipelineRunner(m, PipelineConfig(num_stages=2), tp.BeamConfig(w=64, k=16), None, collect_trace=False,
                   kv_capacity=1024)
r.prefill(prompt)
st = r.stages[0]
n = 16
pre = np.full(n, 512, dtype=np.int32)
bits = np.zeros((n, 1), dtype=np.uint64)
x = torch.randn(n, cfg.hidden, device="cuda")
item = (st.kv, m, x, None, [512] * n, (0, 4), False, list(range(n)), False, (pre, 512, 1, bits))
lib = _lib.lib()
side = torch.cuda.Stream()  # a capturable stream (TP_GRAPH=1 engages on non-default streams)
side.wait_stream(torch.cuda.current_stream())
ctx = torch.cuda.stream(side)
ctx.__enter__()
for mask, label in ((0, "full"), (5, "prep only (GEMM + attention launches skipped)")):
    _lib.check(lib.tp_debug_attn_knob(3, mask))
    for _ in range(20):
        forward_members([[item]])
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    dts = []
    n_calls = 50
    for _ in range(50):  # one call at a time on an idle GPU: no launch-queue back-pressure
        torch.cuda.synchronize()
        t = time.perf_counter()
        forward_members([[item]])
        dts.append(time.perf_counter() - t)
        torch.cuda.synchronize()
    for _ in range(3):  # and the GPU time of one call
        forward_members([[item]])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        forward_members([[item]])
    e1.record()
    torch.cuda.synchronize()
    gpu_us = e0.elapsed_time(e1) * 1e3 / 20
    dt = float(np.median(dts))
    nl = (_lib.launch_count() - l0) / (n_calls + 23)
    torch.cuda.synchronize()
    print(f"{label}: {dt * 1e6:.1f} us host per forward call, {nl:.0f} launches, {gpu_us:.1f} us GPU per call "
          f"(back to back)", flush=True)
_lib.check(lib.tp_debug_attn_knob(3, 0))
