"""Drop-in proof: the UNMODIFIED reference step machine on the B200 path.

The reference package is installed untouched under baseline/_ref (see
DESIGN.md §8; `pip install --no-deps --target baseline/_ref`).  Exactly the
patch INTEGRATION.md §1 gives a treepipe maintainer is applied — the module
globals `treepipe/pipeline.py:35` binds at import (`KvCache`, `forward_tree`,
`sequential_decode`) plus a B200 model object — and the reference's own
`PipelineRunner` (`pipeline.py:155-573`) then drives every step: its
`forward_tree` calls (`:294-301`), `greedy_token` (`:328`), `promote` /
`prune` / `drop_speculative` (`:351-361`) and the payload hand-off
(`:373-439`) all land in libtreepipe_b200.so.

Checked against the reference's own recorded runs (tests/golden): tokens,
hit / flush, every stage's KV keep list and `tree.encode` bytes, bit-exact.
"""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, ListReplay, pipeline_case

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "treepipe")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, REF)
    try:
        mods = {name: importlib.import_module(f"treepipe{name}") for name in ("", ".pipeline")}
    finally:
        sys.path.remove(REF)
    P = mods[".pipeline"]
    saved = {k: getattr(P, k) for k in ("KvCache", "forward_tree", "sequential_decode")}
    import paper_2504_04104_b200.model as B

    # INTEGRATION.md §1, verbatim
    P.KvCache = B.KvCache
    P.forward_tree = B.forward_tree
    P.sequential_decode = B.sequential_decode
    yield mods[""], P
    for k, v in saved.items():
        setattr(P, k, v)


@pytest.mark.parametrize("idx", [0, 1, 2, "c1_paper"])
def test_reference_runner_on_b200(golden, ref, idx):
    treepipe, P = ref
    case = pipeline_case(golden, idx)
    model = tp.init_model(tp.ToyModelConfig(**case["model"]))  # B200 ToyModel (f64 kernels)
    runner = P.PipelineRunner(model, treepipe.PipelineConfig(num_stages=case["stages"]),
                              treepipe.BeamConfig(w=case["w"], k=case["k"]), ListReplay(case["trace"]),
                              collect_trace=False)
    assert all(isinstance(s.kv, tp.model.KvCache) for s in runner.stages)
    runner.prefill(case["prompt"])
    for si, want in enumerate(case["steps"]):
        for s in runner.stages:
            s.kv.last_keep = None
        o = runner.decode_step()
        assert o.verified_token == want["token"], si
        assert o.hit == want["hit"] and o.flush_depth == want["flush_depth"], si
        keeps = [s.kv.last_keep for s in runner.stages]
        assert (keeps if any(k is not None for k in keeps) else None) == want["keeps"], si
        assert treepipe.encode(runner.tree).hex() == want["tree"], si
    assert runner.emitted == case["emitted"] == case["reference"]
    assert runner.metrics().to_json() == case["metrics"]


def test_reference_run_llama_lossless(ref):
    """The reference's own `run()` (`pipeline.py:587-613`: sequential_decode to bind
    the synthetic draft, then decode_step until done) over a B200 Llama-shape
    model: SpecPipe tokens == greedy decode through the same kernels."""
    treepipe, P = ref
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
    model = tp.LlamaModel(cfg, max_nodes=64)
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, 512, 40)]
    want = tp.sequential_decode(model, prompt, 24)
    draft = treepipe.SyntheticDraft(treepipe.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1,
                                                                  seed=3), cfg.vocab)
    res = P.run(model, treepipe.PipelineConfig(num_stages=4), treepipe.BeamConfig(w=8, k=4), draft, prompt, 24)
    assert res.tokens == want
