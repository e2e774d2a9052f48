"""Host cost of the stage-per-GPU step protocol, emulated on one GPU: the bench
workload (7B, 8 stages, w64/k16, paper draft) with one shard model object per
stage (bench.py --gpus 8 placement) on shard streams.  Reports host time per
step by phase and a cProfile of the busiest functions.

    python scripts/host_cross.py [--steps 64] [--profile]
"""
import argparse
import cProfile
import gc
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import draft_cfg, model_cfg  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel  # noqa: E402
from paper_2504_04104_b200.pipeline import (PipelineConfig, PipelineRunner, sequential_decode_staged,  # noqa: E402
                                            split_layers)

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--grouped", type=int, default=1)
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()
cfg = model_cfg(args.model)
stages = 8
splits = split_layers(cfg.layers, stages)
shards = [LlamaModel(cfg, device=0, max_nodes=64, layer_range=(lo, hi), with_embed=(lo == 0),
                     with_head=(hi == cfg.layers)) for lo, hi in splits]  # one shard per stage, all on GPU 0
prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, 512)]
ref = sequential_decode_staged(shards, splits, prompt, 200)
draft = tp.SyntheticDraft(draft_cfg("paper"), cfg.vocab)
draft.bind_reference(tuple(prompt) + tuple(ref))
r = PipelineRunner(shards, PipelineConfig(num_stages=stages, layer_splits=tuple(splits)), tp.BeamConfig(w=64, k=16),
                   draft, collect_trace=False, kv_capacity=2048, check_invariants=False, grouped=bool(args.grouped),
                   shard_streams=True)
r.prefill(prompt)
for _ in range(24):
    r.decode_step()
torch.cuda.synchronize()
r.host_s = {k: 0.0 for k in r.host_s}
gc.collect()
gc.disable()
pr = cProfile.Profile() if args.profile else None
t0 = time.perf_counter()
c0 = time.process_time()
if pr:
    pr.enable()
for _ in range(args.steps):
    r.decode_step()
if pr:
    pr.disable()
wall = time.perf_counter() - t0
cpu = time.process_time() - c0
torch.cuda.synchronize()
gc.enable()
assert r.emitted == ref[: len(r.emitted)]
h = {k: round(v * 1e3 / args.steps, 4) for k, v in r.host_s.items()}
print(f"cross protocol, 8 shards on 1 GPU, grouped={args.grouped}: wall {wall * 1e3 / args.steps:.3f} ms/step, "
      f"process cpu {cpu * 1e3 / args.steps:.3f} ms/step, host phases {h}, "
      f"busy (wall - verify_wait) {wall * 1e3 / args.steps - h['verify_wait']:.3f} ms/step", flush=True)
if pr:
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
