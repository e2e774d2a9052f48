"""Small Llama pipeline run for compute-sanitizer (memcheck / racecheck / synccheck):
exercises grouped GEMMs, the shared-prefix run and per-node tail attention kernels, K3, K4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402

cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
m = tp.LlamaModel(cfg, max_nodes=64)
prompt = [int(t) for t in np.random.default_rng(3).integers(0, 512, 90)]
ref = tp.sequential_decode(m, prompt, 12)
for _ in range(2):
    d = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1, seed=1), 512)
    res = tp.run(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=12, k=4), d, prompt, 10, collect_trace=False)
    assert res.tokens == ref[:10], (res.tokens, ref[:10])
print("sanitize step ok")
