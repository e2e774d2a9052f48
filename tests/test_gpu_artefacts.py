"""Byte-level parity of the on-disk / wire artefacts with files WRITTEN BY THE
UNMODIFIED REFERENCE (tests/golden/make_golden.py `artefacts()`):

* checkpoint (`/root/reference/pkg/src/treepipe/model.py:388-435`): our writer
  produces the reference's bytes for the same config, and the reference's file
  loads into HBM weights equal to the LCG init;
* StepTrace CSV (`pipeline.py:123-152`) and RunMetrics JSON (`:549-573`) of a
  3-stage run: byte-identical CSV, equal metrics, equal tokens;
* draft-trace JSONL (`token_source.py:178-226`) recorded during that run:
  byte-identical, and replaying the reference's file reproduces the run.
"""

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")


def test_checkpoint_bytes_equal_reference(tmp_path):
    model = tp.init_model(tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=11))
    path = str(tmp_path / "ours.bin")
    tp.save_checkpoint(model, path)
    with open(path, "rb") as a, open(os.path.join(GOLDEN, "ref_ckpt_v32_d8_l2_s11.bin"), "rb") as b:
        assert a.read() == b.read()
    back = tp.load_checkpoint(os.path.join(GOLDEN, "ref_ckpt_v32_d8_l2_s11.bin"))
    assert np.array_equal(back.embedding, model.embedding)
    for layer in range(2):
        for k, v in model.layer_weights(layer).items():
            assert np.array_equal(back.layer_weights(layer)[k], v), (layer, k)


def test_trace_csv_metrics_and_draft_trace_equal_reference(tmp_path):
    with open(os.path.join(GOLDEN, "ref_metrics_m3.json")) as fh:
        want = json.load(fh)
    model = tp.init_model(tp.ToyModelConfig(**want["model"]))
    prompt = want["prompt"]
    ref_tokens = tp.sequential_decode(model, prompt, 24)
    rec = tp.RecordingDraft(tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1,
                                                                       seed=9), 48))
    rec.bind_reference(tuple(prompt) + tuple(ref_tokens))
    res = tp.run(model, tp.PipelineConfig(num_stages=want["stages"]), tp.BeamConfig(w=want["w"], k=want["k"]), rec,
                 prompt, 24)
    assert res.tokens == want["tokens"]
    assert res.metrics.to_json() == want["metrics"]
    buf = io.StringIO()
    tp.write_trace_csv(res.trace, buf)
    with open(os.path.join(GOLDEN, "ref_trace_m3.csv"), newline="") as fh:
        assert buf.getvalue() == fh.read()
    ours = str(tmp_path / "draft.jsonl")
    tp.write_trace(rec.records, ours)
    with open(ours, "rb") as a, open(os.path.join(GOLDEN, "ref_draft_m3.jsonl"), "rb") as b:
        assert a.read() == b.read()
    # replaying the reference-written draft trace reproduces the run
    replay = tp.ReplayDraft.from_file(os.path.join(GOLDEN, "ref_draft_m3.jsonl"))
    res2 = tp.run(model, tp.PipelineConfig(num_stages=want["stages"]), tp.BeamConfig(w=want["w"], k=want["k"]),
                  replay, prompt, 24)
    assert res2.tokens == want["tokens"] and res2.metrics.to_json() == want["metrics"]
