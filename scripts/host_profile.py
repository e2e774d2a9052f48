"""cProfile of the host side of decode_step at the bench workload (GPU box)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import model_cfg  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner  # noqa: E402

cfg = model_cfg(sys.argv[1] if len(sys.argv) > 1 else "7b")
m = LlamaModel(cfg, max_nodes=64)
prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, 512)]
ref = tp.sequential_decode(m, prompt, 120)
draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=0), cfg.vocab)
draft.bind_reference(tuple(prompt) + tuple(ref))
r = PipelineRunner(m, PipelineConfig(num_stages=8), tp.BeamConfig(w=64, k=16), draft, collect_trace=False,
                   kv_capacity=2048, check_invariants=False)
r.prefill(prompt)
for _ in range(16):
    r.decode_step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(40):
    r.decode_step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(45)
