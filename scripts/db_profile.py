"""Host profile of SpecPipe-DB steady-state ticks (13B, 8 stages, width 64):
wall vs GPU time per tick and a cProfile of the host side.

    python scripts/db_profile.py [--batch 16] [--ticks 20]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import model_cfg  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="13b")
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ticks", type=int, default=20)
ap.add_argument("--ncu-window", type=int, default=0, help="only run N ticks between cudaProfilerStart/Stop, then exit")
args = ap.parse_args()
cfg = model_cfg(args.model)
m = LlamaModel(cfg, max_nodes=64)
V = cfg.vocab
new_tokens = 64
reqs = [tp.Request(i, 0, tuple(int(t) for t in np.random.default_rng([0, i + 1]).integers(0, V, 512)), new_tokens)
        for i in range(args.batch)]
refs = dict(enumerate(tp.sequential_decode_batch(m, [list(r.prompt) for r in reqs], new_tokens)))
bcfg = tp.BatchConfig(max_batch=args.batch, total_width=64, k=16, draft=tp.SyntheticDraftConfig(seed=0),
                      check_isolation_every_tick=False)
sched = tp.BatchScheduler(m, tp.PipelineConfig(num_stages=8), bcfg, references=refs, combined=True)
for r in reqs:
    sched.submit(r)
sched.queue.sort(key=lambda r: (r.arrival_tick, r.request_id))
for _ in range(6):
    sched.tick()
torch.cuda.synchronize()
if args.ncu_window:
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.ncu_window):
        sched.tick()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sys.exit(0)
walls, gpus = [], []
for _ in range(args.ticks):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    sched.tick()
    e1.record()
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t) * 1e3)
    gpus.append(e0.elapsed_time(e1))
print(f"batch {args.batch}: wall {np.mean(walls):.3f} ms/tick, GPU span {np.mean(gpus):.3f} ms/tick (synchronised ticks)")
# host phases of an unsynchronised tick (wrappers around the tick's parts)
import paper_2504_04104_b200.batching as B  # noqa: E402
import paper_2504_04104_b200.model as M  # noqa: E402

acc = {}


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
    return w


sched._combined_launch = timed("combined_launch", sched._combined_launch)
sched._combined_wait = timed("combined_wait", sched._combined_wait)
for slot in sched.active:
    slot.runner.draft_children = timed("draft_children", slot.runner.draft_children)
    slot.runner.step = timed("step", slot.runner.step)
M._launch_restrict = timed("flush_restrict", M._launch_restrict)
M._launch_rows = timed("flush_rows", M._launch_rows)
import gc  # noqa: E402

gc.collect()
gc.disable()
t = time.perf_counter()
for _ in range(args.ticks):
    sched.tick()
torch.cuda.synchronize()
tot = time.perf_counter() - t
gc.enable()
print(f"unsynchronised: {tot * 1e3 / args.ticks:.3f} ms/tick; host phases ms/tick:",
      {k: round(v * 1e3 / args.ticks, 3) for k, v in acc.items()})
pr = cProfile.Profile()
pr.enable()
for _ in range(args.ticks):
    sched.tick()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
