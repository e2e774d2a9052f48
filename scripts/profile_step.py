"""Profile window for ncu: N SpecPipe steps of the bench workload between
cudaProfilerStart/Stop (run under `ncu --profile-from-start off ...`).

    python scripts/profile_step.py [--model 7b] [--steps 4] [--warmup 16]
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
from paper_2504_04104_b200.model import LlamaModel  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=16)
ap.add_argument("--prompt-len", type=int, default=512)
ap.add_argument("--timeline", action="store_true", help="print host-side timing of each phase")
ap.add_argument("--draft-model", default="68m", choices=["68m", "none"], help="draft model forward each step (bench default)")
args = ap.parse_args()

cfg = model_cfg(args.model)
m = LlamaModel(cfg, max_nodes=64)
prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, args.prompt_len)]
ref = tp.sequential_decode(m, prompt, args.warmup + args.steps + 24)
draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=0), cfg.vocab)
draft.bind_reference(tuple(prompt) + tuple(ref))
dm = LlamaModel(tp.LlamaConfig.llama_68m(), max_nodes=64) if args.draft_model == "68m" else None
r = PipelineRunner(m, PipelineConfig(num_stages=8), tp.BeamConfig(w=64, k=16), draft, collect_trace=False,
                   kv_capacity=2048, check_invariants=False, draft_model=dm)
r.prefill(prompt)
for _ in range(args.warmup):
    r.decode_step()
torch.cuda.synchronize()
from paper_2504_04104_b200 import _lib  # noqa: E402

_lib.profile_enable(True)  # per-launch algorithmic bytes of every K2 launch in the window
torch.cuda.profiler.start()
t0 = time.perf_counter()
for _ in range(args.steps):
    r.decode_step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
_lib.profile_enable(False)
ms, by, nl = _lib.profile_read()
print(f"gemm_launches={nl} algorithmic_bytes_total={by:.0f} algorithmic_bytes_per_launch={by / max(1, nl):.0f}")
dt = (time.perf_counter() - t0) * 1e3 / args.steps
print(f"steps={args.steps} wall/step={dt:.3f} ms resident={[len(s.resident) if s.resident else 0 for s in r.stages]}")
