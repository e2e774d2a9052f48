"""Kernel-time breakdown of the SpecPipe-DB admission prefill (13B shape, 8
stages, B requests x prompt_len rows through ``prefill_requests``) at a given
``max_nodes`` (rows per combined forward).  GPU box only.

    python scripts/prefill_profile.py [--batch 8] [--max-nodes 256]   (K2 takes at most 256 rows)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import model_cfg  # noqa: E402
from paper_2504_04104_b200.batching import prefill_requests  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineRunner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="13b")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--prompt-len", type=int, default=512)
ap.add_argument("--max-nodes", type=int, default=256)
args = ap.parse_args()
cfg = model_cfg(args.model)
m = LlamaModel(cfg, max_nodes=args.max_nodes)
V = cfg.vocab
prompts = [[int(t) for t in np.random.default_rng([0, i + 1]).integers(0, V, args.prompt_len)]
           for i in range(args.batch)]


def runners():
    return [PipelineRunner(m, tp.PipelineConfig(num_stages=8), tp.BeamConfig(w=8, k=4), None, collect_trace=False,
                           kv_capacity=args.prompt_len + 64, check_invariants=False) for _ in prompts]


rs = runners()
prefill_requests(rs, prompts)  # warm-up (workspace growth, first-use costs)
torch.cuda.synchronize()
for r in rs:
    r.release()
rs = runners()
torch.cuda.synchronize()
t = time.perf_counter()
prefill_requests(rs, prompts)
torch.cuda.synchronize()
wall = time.perf_counter() - t
rows = args.batch * args.prompt_len
print(f"batch {args.batch} x {args.prompt_len} rows, max_nodes {args.max_nodes}: {wall * 1e3:.1f} ms "
      f"({wall * 1e6 / rows:.1f} us/row)")
for r in rs:
    r.release()
rs = runners()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    prefill_requests(rs, prompts)
    torch.cuda.synchronize()
acc = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0][:60]
        a = acc.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in acc.values())
print(f"kernel time {tot / 1e3:.1f} ms (profiled run)")
for name, (n, us) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {us / 1e3:9.2f} ms  {n:6d}  {name}")
