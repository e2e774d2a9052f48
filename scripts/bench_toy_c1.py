"""BASELINE config 1 (the reference's CPU demo): ToyModel V=64, d=256, L=4
(float64, exactly the reference architecture), 2 stages, beam w=4/k=4 (CLI
defaults) and w=64/k=16, SyntheticDraft paper defaults, greedy, 128-token
prompt.  Reports wall-clock TBT of `run()` (host control included).

    python scripts/bench_toy_c1.py            # B200 path (this package)
    python scripts/bench_toy_c1.py --reference  # unmodified reference (CPU; build container only)
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reference", action="store_true")
ap.add_argument("--tokens", type=int, default=64)
args = ap.parse_args()
if args.reference:
    sys.path.insert(0, "/root/reference/pkg/src")
    import treepipe as tp  # noqa: E402
else:
    import paper_2504_04104_b200 as tp  # noqa: E402

cfg = tp.ToyModelConfig(vocab=64, hidden=256, layers=4, seed=0)
model = tp.init_model(cfg)
prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, 64, 128)]
for w, k in ((4, 4), (64, 16)):
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=0), 64)
    t0 = time.perf_counter()
    res = tp.run(model, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=w, k=k), draft, prompt, args.tokens,
                 collect_trace=False) if not args.reference else \
        tp.run(model, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=w, k=k), draft, prompt, args.tokens)
    wall = time.perf_counter() - t0
    # run() includes the oracle decode that binds the draft (reference pipeline.py:599-602)
    t1 = time.perf_counter()
    tp.sequential_decode(model, prompt, args.tokens)
    seq = time.perf_counter() - t1
    print(json.dumps({"impl": "reference-cpu" if args.reference else "b200", "config": "C1 toy V64 d256 L4, 2 stages",
                      "w": w, "k": k, "tokens": len(res.tokens), "run_wall_s": round(wall, 4),
                      "tbt_ms_per_token_excl_binding": round((wall - seq) * 1e3 / len(res.tokens), 4),
                      "sequential_decode_ms_per_token": round(seq * 1e3 / args.tokens, 4),
                      "steps_per_token": round(res.metrics.steps_per_token, 4), "tokens_head": res.tokens[:8]}),
          flush=True)
