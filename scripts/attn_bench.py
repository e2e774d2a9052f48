"""K1 in isolation, in situ: the grouped phase-1 forward of 7 same-device 7B
stages (bench mean node counts, 512-row prefix + ancestor chains) with the
GEMMs and RMSNorms skipped (diagnostic knob 3, WRONG results), minus the same
forward with attention skipped too = attention time per forward; / layers =
per layer slot.  TP_ATTN_DEBUG=1 / 2 (skip tail / run kernel) splits it.

    python scripts/attn_bench.py [--prefix 512] [--n 45,35,29,23,17,11,3] [--run 4]
"""
import argparse
import json
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
ap.add_argument("--run", type=int, default=0)
args = ap.parse_args()
cfg = model_cfg(args.model)
m = LlamaModel(cfg, max_nodes=64)
ns = [int(x) for x in args.n.split(",")]
depth = 12
prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab, args.prefix + depth)]
r = PipelineRunner(m, PipelineConfig(num_stages=len(ns) + 1), tp.BeamConfig(w=64, k=16), None, collect_trace=False,
                   kv_capacity=max(2048, args.prefix + 256))
r.prefill(prompt)
rng = np.random.default_rng(2)
items = []
for s, n in zip(r.stages, ns):
    d = rng.integers(0, depth, n)
    pre = np.full(n, args.prefix, dtype=np.int32)
    bits = ((np.uint64(1) << d.astype(np.uint64)) - np.uint64(1)).reshape(n, 1).astype(np.uint64)
    x = torch.randn(n, cfg.hidden, device="cuda") * 0.5  # fp32 residual-stream rows
    items.append((s.kv, m, x, None, (args.prefix + d).tolist(), s.layer_range, False, list(range(n)), False,
                  (pre, args.prefix, 1, bits)))
lib = _lib.lib()
if args.run:
    _lib.check(lib.tp_debug_attn_knob(1, args.run))
layers = cfg.layers // (len(ns) + 1)


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


out = {"prefix": args.prefix, "n": ns, "attn_debug": os.environ.get("TP_ATTN_DEBUG", "0")}
for name, members in (("group", [[it] for it in items]), ("single", [[items[-1]]])):
    a = timed(members, 6)  # attention + prep
    b = timed(members, 7)  # prep only
    out[name + "_us_per_slot"] = round((a - b) / layers, 2)
print(json.dumps(out), flush=True)
