import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_04104_b200 as tp
from paper_2504_04104_b200.model import LlamaConfig, LlamaModel
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner

cfg = LlamaConfig(vocab=512, hidden=256, layers=8, heads=2, kv_heads=1, ffn=512)
m = LlamaModel(cfg, max_nodes=64)
prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, 100)]
ref = tp.sequential_decode(m, prompt, 80)
pcfg = PipelineConfig(num_stages=8)
beam = tp.BeamConfig(w=64, k=16)
def fresh(d):
    r = PipelineRunner(m, pcfg, beam, d, collect_trace=False, kv_capacity=2048, check_invariants=True)
    r.prefill(prompt); return r
d = tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=0), cfg.vocab); d.bind_reference(tuple(prompt)+tuple(ref))
a = fresh(d); a.children_log = []
trees_a = []
for i in range(40):
    a.decode_step(); trees_a.append(tp.encode(a.tree))
print("e2e emitted", a.emitted[:10], a.emitted == ref[:len(a.emitted)])
b = fresh(None)
for i, ch in enumerate(a.children_log):
    try:
        b.step(ch)
    except Exception as e:
        print("replay failed at", i, repr(e)); break
    if tp.encode(b.tree) != trees_a[i]:
        print("tree diverged at step", i, "tokens", a.emitted[:len(b.emitted)] == b.emitted, b.emitted[-3:], a.emitted[len(b.emitted)-3:len(b.emitted)])
        break
else:
    print("replay identical", b.emitted == a.emitted)
