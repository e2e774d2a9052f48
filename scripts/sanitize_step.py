"""Small Llama pipeline runs for compute-sanitizer (memcheck / racecheck / synccheck):
grouped GEMMs (stream-K fix-up, reducer queue), the shared-prefix run kernel in both
CTA shapes (row-parallel and chunk-parallel), the per-node and GQA tails (early
chunks before griddepcontrol.wait), K3, K4.  A 600-token prompt gives 9 canonical
chunks: two full runs of 4 plus a partial one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402

configs = {"mha": (2, 1), "gqa": (4, 1)}  # MHA-like per-node tail, GQA tail (group 4)
small = os.environ.get("TP_SANITIZE_SMALL") == "1"  # racecheck of the GQA config: a shorter decode
for heads, kv in [configs[a] for a in (sys.argv[1:] or configs)]:
    cfg = tp.LlamaConfig(vocab=512, hidden=128 * heads, layers=4, heads=heads, kv_heads=kv, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 512, 300 if small else 600)]
    n_tok = 4 if small else 10
    ref = tp.sequential_decode(m, prompt, n_tok + 2)
    d = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1, seed=1), 512)
    res = tp.run(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=6 if small else 12, k=4), d, prompt, n_tok,
                 collect_trace=False)
    assert res.tokens == ref[:n_tok], (res.tokens, ref[:n_tok])
print("sanitize step ok")
