"""Small Llama pipeline runs for compute-sanitizer (memcheck / racecheck / synccheck):
grouped GEMMs (stream-K fix-up, reducer queue), the shared-prefix run kernel in both
CTA shapes (row-parallel and chunk-parallel), the per-node and GQA tails (early
chunks before griddepcontrol.wait), K3, K4.  A 600-token prompt gives 9 canonical
chunks: two full runs of 4 plus a partial one.  "draft" adds a draft model fused into the
verify stage's launches (per-member GEMM plans, mixed-model attention / norm groups) and
the top-k kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402

configs = {"mha": (2, 1), "gqa": (4, 1), "draft": (2, 1)}  # MHA-like tail, GQA tail (group 4), + draft model
small = os.environ.get("TP_SANITIZE_SMALL") == "1"  # racecheck of the GQA config: a shorter decode
for name in sys.argv[1:] or list(configs):
    heads, kv = configs[name]
    cfg = tp.LlamaConfig(vocab=512, hidden=128 * heads, layers=4, heads=heads, kv_heads=kv, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 512, 300 if small else 600)]
    n_tok = 4 if small else 10
    ref = tp.sequential_decode(m, prompt, n_tok + 2)
    d = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1, seed=1), 512)
    if name == "draft":  # the draft model fused into the verify stage's launches (heterogeneous groups) + top-k
        from paper_2504_04104_b200.pipeline import PipelineRunner

        dm = tp.LlamaModel(tp.LlamaConfig(vocab=512, hidden=256, layers=1, heads=2, kv_heads=2, ffn=384, seed=5),
                           max_nodes=64)
        d.bind_reference(tuple(prompt) + tuple(ref))
        r = PipelineRunner(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=6 if small else 12, k=4), d,
                           collect_trace=False, draft_model=dm)
        r.prefill(prompt)
        while len(r.emitted) < n_tok:
            r.decode_step()
        assert r.emitted[:n_tok] == ref[:n_tok]
        continue
    res = tp.run(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=6 if small else 12, k=4), d, prompt, n_tok,
                 collect_trace=False)
    assert res.tokens == ref[:n_tok], (res.tokens, ref[:n_tok])
print("sanitize step ok")
