"""K3 driven by the device-resident verification result (tp_prune_device).

The keep lists the device derives from K4's token and the packed tree rows
(ballot + warp prefix sum) must equal the reference's `_restrict` keep lists
(pipeline.py:341-361, model.py:184) — checked against the reference's own
recorded runs — and a pipeline pruned on the device must stay bit-identical,
step by step, to the host-keep-list path.
"""

import numpy as np
import pytest
import torch

from conftest import PIPE_CASES, ListReplay, pipeline_case

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200 import pipeline as pl  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineRunner  # noqa: E402


def device_lists(bufs):
    out = []
    for b in bufs:
        v = b.cpu().numpy()
        out.append(v)
    return out


@pytest.mark.parametrize("idx", PIPE_CASES)
def test_device_keep_lists_equal_reference(golden, idx, monkeypatch):
    monkeypatch.setattr(pl, "_DEVICE_PRUNE", True)
    case = pipeline_case(golden, idx)
    model = tp.init_model(tp.ToyModelConfig(**case["model"]))
    runner = PipelineRunner(model, tp.PipelineConfig(num_stages=case["stages"]),
                            tp.BeamConfig(w=case["w"], k=case["k"]), ListReplay(case["trace"]))
    runner.capture_device_keeps = []
    runner.prefill(case["prompt"])
    checked = 0
    for si, want in enumerate(case["steps"]):
        n_cap = len(runner.capture_device_keeps)
        o = runner.decode_step()
        assert o.verified_token == want["token"] and runner.last_keeps == want["keeps"], si
        assert tp.encode(runner.tree).hex() == want["tree"], si
        if len(runner.capture_device_keeps) > n_cap:
            bufs = runner.capture_device_keeps[-1]
            for stage_i, (buf, keep) in enumerate(zip(device_lists(bufs), want["keeps"])):
                ns = int(buf[0])
                # device list holds the kept speculative rows; the reference list = prefix + those rows
                spec = [int(r) for r in buf[2:2 + ns]]
                P = len(keep) - ns
                assert keep == list(range(P)) + spec, (si, stage_i)
                checked += 1
    assert runner.emitted == case["emitted"]
    assert checked > 0


@pytest.mark.parametrize("stages,w,k,miss", [(4, 8, 4, 0.1), (8, 16, 4, 0.3), (3, 5, 3, 0.0)])
def test_device_prune_bitwise_equals_host_prune(stages, w, k, miss, monkeypatch):
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=stages, heads=2, kv_heads=1, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 512, 70)]
    ref = tp.sequential_decode(m, prompt, 40 + 3 * stages)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=miss, seed=7), 512)
    draft.bind_reference(tuple(prompt) + tuple(ref))
    monkeypatch.setattr(pl, "_DEVICE_PRUNE", False)
    rec = PipelineRunner(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=w, k=k), draft,
                         collect_trace=False)
    rec.children_log = []
    rec.prefill(prompt)
    while len(rec.emitted) < 24:
        rec.decode_step()
    runs = {}
    for dev in (False, True):
        monkeypatch.setattr(pl, "_DEVICE_PRUNE", dev)
        r = PipelineRunner(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=w, k=k), None,
                           collect_trace=False)
        r.prefill(prompt)
        outs, keeps = [], []
        for ch in rec.children_log:
            r.launch_compute()
            outs.append([None if s.out is None else s.out.cpu().clone() for s in r.stages])
            r.step(ch)
            keeps.append(r.last_keeps)
        kv = [[s.kv.keys[s.layer_range[0]] for s in r.stages]]
        runs[dev] = (outs, keeps, list(r.emitted), kv)
    assert runs[True][2] == runs[False][2] == rec.emitted == ref[: len(rec.emitted)]
    assert runs[True][1] == runs[False][1]
    for step, (a, b) in enumerate(zip(runs[True][0], runs[False][0])):
        for s, (x, y) in enumerate(zip(a, b)):
            assert (x is None) == (y is None), (step, s)
            if x is not None:
                assert torch.equal(x, y), (step, s)
    for x, y in zip(runs[True][3][0], runs[False][3][0]):
        assert np.array_equal(x, y)
