"""Marginal cost of each kernel class inside one grouped phase-1 forward (PDL
chain intact): 7 same-device stages of the 7B bench at its mean per-stage node
counts, 512-token prefix + tree ancestors, timed with CUDA events; then the
same with attention / RMSNorm / GEMMs skipped (diagnostic knob, WRONG results).

    python scripts/ablate_fwd.py [--iters 50] [--n 45,35,29,23,17,11,3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import model_cfg  # noqa: E402
from paper_2504_04104_b200 import _lib  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel, forward_members  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--prefix", type=int, default=512)
ap.add_argument("--n", default="45,35,29,23,17,11,3")
ap.add_argument("--run", type=int, default=0, help="attention chunks per run (knob 1; 0 = built-in)")
ap.add_argument("--masks", default="1,4,7")
ap.add_argument("--timeline", action="store_true", help="per kernel-class timeline of each forward (CUDA events)")
ap.add_argument("--sib", type=float, default=0.0, help="mean sibling-group size (0: every node its own chain)")
args = ap.parse_args()
cfg = model_cfg(args.model)
m = LlamaModel(cfg, max_nodes=64)
ns = [int(x) for x in args.n.split(",")]
depth = 12  # ancestors per node < 16 (the attention suffix window)
prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab, args.prefix + depth)]
r = PipelineRunner(m, PipelineConfig(num_stages=len(ns) + 1), tp.BeamConfig(w=64, k=16), None, collect_trace=False,
                   kv_capacity=2048)
r.prefill(prompt)
rng = np.random.default_rng(2)
items = []
for s, n in zip(r.stages, ns):
    d = rng.integers(0, depth, n)  # node i: ancestors = rows prefix .. prefix+d_i-1 (a chain), then itself
    if args.sib > 0:  # consecutive siblings share the parent's chain (groups ~ geometric, mean args.sib)
        i = 0
        while i < n:
            gsz = int(min(16, n - i, rng.geometric(1.0 / args.sib)))
            d[i : i + gsz] = d[i]
            i += gsz
    pre = np.full(n, args.prefix, dtype=np.int32)
    bits = ((np.uint64(1) << d.astype(np.uint64)) - np.uint64(1)).reshape(n, 1).astype(np.uint64)
    x = torch.randn(n, cfg.hidden, device="cuda") * 0.5  # fp32 residual-stream rows
    items.append((s.kv, m, x, None, (args.prefix + d).tolist(), s.layer_range, False, list(range(n)), False,
                  (pre, args.prefix, 1, bits)))
lib = _lib.lib()
if args.run:
    _lib.check(lib.tp_debug_attn_knob(1, args.run))


def timed(members, mask):
    _lib.check(lib.tp_debug_attn_knob(3, mask))
    for _ in range(3):
        forward_members(members)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        forward_members(members)
    e1.record()
    torch.cuda.synchronize()
    _lib.check(lib.tp_debug_attn_knob(3, 0))
    return e0.elapsed_time(e1) * 1e3 / args.iters


if args.timeline:
    for name, members in (("group", [[it] for it in items]), ("single", [[items[-1]]])):
        for _ in range(3):
            forward_members(members)
        torch.cuda.synchronize()
        _lib.timeline_enable(True)
        _lib.timeline_read()
        for _ in range(args.iters):
            forward_members(members)
        torch.cuda.synchronize()
        _lib.timeline_enable(False)
        tl = {k: round(v * 1e3 / args.iters, 1) for k, v in sorted(_lib.timeline_read().items(), key=lambda kv: -kv[1])}
        print(f"{name} timeline us/forward: {tl} total {round(sum(tl.values()), 1)}", flush=True)

labels = {0: "full", 1: "-attention", 2: "(no-op: norm folded)", 3: "-attention", 4: "-gemm", 7: "host+prep only"}
for name, members in (("group of %d" % len(ns), [[it] for it in items]), ("single (n=1)", [[items[-1]]])):
    base = timed(members, 0)
    print(f"{name}: full forward {base:8.1f} us", flush=True)
    for mask in [int(x) for x in args.masks.split(",") if x]:
        t = timed(members, mask)
        print(f"  {labels[mask]:15s} {t:8.1f} us   (saves {base - t:7.1f} us)", flush=True)
