"""SpecPipe-DB (batching.py mirror): host logic on CPU; the combined ragged GPU
step on the B200 (outputs equal each request's solo greedy decode)."""

import json

import numpy as np
import pytest

import paper_2504_04104_b200 as tp
from paper_2504_04104_b200.batching import RaggedBatch, check_isolation, load_workload, split_width
from paper_2504_04104_b200.errors import ConfigError, InvariantViolation, TraceParseError


def test_split_width_matches_reference_rule():
    assert split_width(8, 3) == [3, 3, 2]
    assert split_width(64, 64) == [1] * 64
    assert split_width(4, 8) == [1] * 8  # floor of 1 per slot (batching.py:142-147)
    assert split_width(5, 0) == []


def test_check_isolation_rejects_cross_request():
    mask = np.eye(2, dtype=bool)
    mask[1, 0] = True
    with pytest.raises(InvariantViolation):
        check_isolation(RaggedBatch((0, 1, 2), (0, 1), (10, 11), mask))
    check_isolation(RaggedBatch((0, 1, 2), (0, 1), (10, 11), np.eye(2, dtype=bool)))


def test_load_workload(tmp_path):
    p = tmp_path / "w.jsonl"
    p.write_text(json.dumps({"arrival_step": 0, "prompt_tokens": 5, "max_new_tokens": 3}) + "\n\n"
                 + json.dumps({"arrival_step": 2, "prompt_tokens": [1, 2], "max_new_tokens": 1}) + "\n")
    reqs = load_workload(str(p), 64, seed=3)
    assert [r.request_id for r in reqs] == [0, 1]
    want = tuple(int(t) for t in np.random.default_rng([3, 1]).integers(0, 64, size=5))
    assert reqs[0].prompt == want and reqs[1].prompt == (1, 2) and reqs[1].arrival_tick == 2
    p.write_text("{not json}\n")
    with pytest.raises(TraceParseError):
        load_workload(str(p), 64)
    with pytest.raises(ConfigError):
        tp.BatchConfig(max_batch=0)


@pytest.mark.gpu
@pytest.mark.parametrize("max_batch", [1, 2, 4])
def test_toy_serve_outputs_equal_solo_oracle(max_batch):
    from oracle.toy import ToyOracle, greedy_continuation

    model = tp.init_model(tp.ToyModelConfig(vocab=64, hidden=16, layers=4, seed=0))
    rng = np.random.default_rng(7)
    reqs = [tp.Request(i, int(i // 2), tuple(int(t) for t in rng.integers(0, 64, 6)), 8) for i in range(5)]
    metrics, slots = tp.serve(model, tp.PipelineConfig(num_stages=2),
                              tp.BatchConfig(max_batch=max_batch, total_width=8, k=4), reqs)
    oracle = ToyOracle(64, 16, 4, 0)
    assert metrics.completed == 5
    for s in slots:
        assert s.runner.emitted[: s.request.max_new_tokens] == greedy_continuation(oracle, list(s.request.prompt),
                                                                                    s.request.max_new_tokens)


@pytest.mark.gpu
def test_sequential_decode_batch_equals_solo():
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    rng = np.random.default_rng(5)
    prompts = [[int(t) for t in rng.integers(0, 512, n)] for n in (7, 30, 65, 12)]
    got = tp.sequential_decode_batch(m, prompts, 12)
    for p, g in zip(prompts, got):
        assert g == tp.sequential_decode(m, p, 12)


@pytest.mark.gpu
@pytest.mark.parametrize("stages,max_batch", [(4, 3), (2, 5), (8, 12)])
def test_llama_combined_tick_equals_solo(stages, max_batch):
    """The combined ragged step (one launch sequence per tick for all requests)
    emits each request's own greedy continuation, identical to uncombined stepping.
    (8, 12): 96 caches per tick, so the deferred KV pruning and row filters of a
    tick exceed one 64-set launch and are split."""
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=max(4, stages), heads=2, kv_heads=1, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    rng = np.random.default_rng(11)
    reqs = [tp.Request(i, int(rng.integers(0, 3)), tuple(int(t) for t in rng.integers(0, 512, 9 + 7 * i)), 10)
            for i in range(max(6, max_batch))]
    refs = dict(enumerate(tp.sequential_decode_batch(m, [list(r.prompt) for r in reqs], 10)))
    out = {}
    for combined in (True, False):
        bcfg = tp.BatchConfig(max_batch=max_batch, total_width=12, k=4,
                              draft=tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=3))
        metrics, slots = tp.serve(m, tp.PipelineConfig(num_stages=stages), bcfg, reqs, references=refs,
                                  combined=combined)
        assert metrics.completed == len(reqs)
        out[combined] = {s.request.request_id: s.runner.emitted[:10] for s in slots}
        for s in slots:
            assert s.runner.emitted[:10] == tp.sequential_decode(m, list(s.request.prompt), 10)
    assert out[True] == out[False]


@pytest.mark.gpu
def test_prefill_requests_bitwise_equal_solo_prefill():
    """Batched admission (prefill_requests: ragged combined forwards, rows shared
    between requests up to max_nodes per call) leaves every stage cache and the
    root output bit-identical to each request's own PipelineRunner.prefill."""
    import torch

    from paper_2504_04104_b200.batching import prefill_requests
    from paper_2504_04104_b200.pipeline import PipelineRunner

    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
    model = tp.LlamaModel(cfg, max_nodes=96)
    rng = np.random.default_rng(6)
    prompts = [[int(t) for t in rng.integers(0, 512, n)] for n in (7, 130, 64, 1, 201)]
    pcfg = tp.PipelineConfig(num_stages=4)
    beam = tp.BeamConfig(w=4, k=2)
    together = [PipelineRunner(model, pcfg, beam, None, collect_trace=False) for _ in prompts]
    prefill_requests(together, prompts)
    for r, p in zip(together, prompts):
        solo = PipelineRunner(model, pcfg, beam, None, collect_trace=False)
        solo.prefill(p)
        assert r.verified == solo.verified and r.tree.tokens.tolist() == solo.tree.tokens.tolist()
        for a, b in zip(r.stages, solo.stages):
            assert a.kv.uids == b.kv.uids and a.kv.positions == b.kv.positions
            lo = a.layer_range[0]
            assert np.array_equal(a.kv.keys[lo], b.kv.keys[lo]) and np.array_equal(a.kv.values[lo], b.kv.values[lo])
    torch.cuda.synchronize()
