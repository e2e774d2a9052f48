"""Step-machine semantics of the reference's pipeline tests on the B200 path
(`/root/reference/pkg/tests/test_pipeline.py:193-232` stalls and replay
exhaustion; checkpoint round trip `test_model.py:142-161`; trace CSV
`test_pipeline.py:272-294`), checked against the CPU step-machine oracle
(oracle/pipeline.py, pinned to the reference's dumps) where it applies."""

import io

import numpy as np
import pytest

from oracle.pipeline import OracleRunner
from oracle.toy import ToyOracle, greedy_continuation

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200.errors import SourceUnavailable  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineRunner  # noqa: E402

CFG = dict(vocab=48, hidden=8, layers=4, seed=3)


def make_draft(miss_prob=0.05, seed=0):
    top1 = min(0.7, 1.0 - miss_prob)
    return tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=top1, rank_decay=0.5, miss_prob=miss_prob, seed=seed),
                             CFG["vocab"])


class FlakySource:
    """Fails every third call; otherwise defers to a synthetic draft (reference test double)."""

    def __init__(self, inner):
        self.inner = inner
        self.calls = 0

    def bind_reference(self, seq):
        self.inner.bind_reference(seq)

    def propose(self, context, k, *, step=0, frontier_node=0):
        self.calls += 1
        if self.calls % 3 == 0:
            raise SourceUnavailable("transient outage")
        return self.inner.propose(context, k, step=step, frontier_node=frontier_node)


def test_stalls_lossless_and_bit_exact_vs_oracle():
    model = tp.init_model(tp.ToyModelConfig(**CFG))
    oracle = ToyOracle(CFG["vocab"], CFG["hidden"], CFG["layers"], CFG["seed"])
    want = greedy_continuation(oracle, [3, 3], 16)
    res = tp.run(model, tp.PipelineConfig(num_stages=3), tp.BeamConfig(w=2, k=2), FlakySource(make_draft()), [3, 3],
                 16)
    assert res.tokens == want
    assert res.metrics.stalls > 0
    # step by step against the oracle step machine fed by an identical flaky source
    d_gpu, d_cpu = FlakySource(make_draft()), FlakySource(make_draft())
    for d in (d_gpu, d_cpu):
        d.bind_reference((3, 3) + tuple(want))
    runner = PipelineRunner(model, tp.PipelineConfig(num_stages=3), tp.BeamConfig(w=2, k=2), d_gpu)
    orc = OracleRunner(oracle, 3, 2, 2, d_cpu)
    runner.prefill([3, 3])
    orc.prefill([3, 3])
    stalls = 0
    while len(runner.emitted) < 16:
        out = runner.decode_step()
        rec = orc.decode_step()
        stalls += out.stalled
        assert out.verified_token == rec["token"]
        assert out.hit == rec["hit"]
        assert runner.last_keeps == rec["keeps"]
        assert tp.encode(runner.tree) == rec["tree"]
    assert stalls > 0


def test_replay_exhaustion_stops_cleanly(tmp_path):
    model = tp.init_model(tp.ToyModelConfig(**CFG))
    recorder = tp.RecordingDraft(make_draft())
    full = tp.run(model, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=2, k=2), recorder, [1, 2], 16)
    path = tmp_path / "trace.jsonl"
    tp.write_trace(recorder.records[:10], str(path))
    partial = tp.run(model, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=2, k=2),
                     tp.ReplayDraft.from_file(str(path)), [1, 2], 16)
    assert 0 < len(partial.tokens) < 16
    assert partial.tokens == full.tokens[: len(partial.tokens)]


def test_checkpoint_round_trip(tmp_path):
    model = tp.init_model(tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=5))
    path = str(tmp_path / "m.ckpt")
    tp.save_checkpoint(model, path)
    back = tp.load_checkpoint(path)
    assert back.cfg == model.cfg
    np.testing.assert_array_equal(back.embedding, model.embedding)
    for layer in range(2):
        for name, w in model.layer_weights(layer).items():
            np.testing.assert_array_equal(back.layer_weights(layer)[name], w)
    assert tp.sequential_decode(back, [1, 2, 3], 6) == tp.sequential_decode(model, [1, 2, 3], 6)
    with open(path, "ab") as fh:
        fh.write(b"\\0")
    with pytest.raises(tp.ShapeError):
        tp.load_checkpoint(path)


def test_trace_csv_schema():
    model = tp.init_model(tp.ToyModelConfig(**CFG))
    res = tp.run(model, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=2, k=2), make_draft(), [1, 2], 6)
    buf = io.StringIO()
    tp.write_trace_csv(res.trace, buf)
    lines = buf.getvalue().strip().splitlines()
    assert lines[0] == "step,stage,phase,start_ms,end_ms,resident_nodes,hit,flush"
    phases = {row["phase"] for row in res.trace}
    assert phases <= {"compute", "prune", "transmit", "idle"} and "compute" in phases
    assert all(r["end_ms"] >= r["start_ms"] for r in res.trace)


def test_llama_stalls_lossless():
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
    m = tp.LlamaModel(cfg, max_nodes=64)
    prompt = [5, 6, 7, 8, 9]
    want = tp.sequential_decode(m, prompt, 20)
    inner = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=2), 512)
    res = tp.run(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=6, k=3), FlakySource(inner), prompt, 20,
                 collect_trace=False)
    assert res.tokens == want
    assert res.metrics.stalls > 0


@pytest.mark.gpu
def test_k4_argmax_first_max_nan_and_child_match():
    """K4 semantics on crafted logits, against numpy (the reference's greedy_token
    is np.argmax: first maximum, a NaN counts as the maximum and the first NaN
    wins; the matched child is the first level-1 node with that token,
    `pipeline.py:333-339`): ties, NaN, duplicate child tokens, >1024 children,
    vocab sizes that are not multiples of the block, and the per-row kernel."""
    import ctypes as C

    import torch

    from paper_2504_04104_b200 import _lib

    lib = _lib.lib()
    rng = np.random.default_rng(7)

    def match(lg, children):
        t = torch.from_numpy(lg).cuda()
        out = np.zeros(2, dtype=np.int32)
        ch = np.asarray(children, dtype=np.int32)
        _lib.check(lib.tp_debug_argmax(0, C.c_void_p(t.data_ptr()), int(lg.dtype == np.float64), lg.size, 1,
                                       ch.ctypes.data, ch.size, out.ctypes.data))
        return int(out[0]), int(out[1])

    for vocab in (1, 7, 1000, 32000, 50257):
        for dtype in (np.float32, np.float64):
            lg = rng.standard_normal(vocab).astype(dtype)
            if vocab > 10:
                lg[vocab // 3] = lg[vocab // 2] = lg[-1] = lg.max() + 1  # three-way tie: lowest id wins
            ref = int(np.argmax(lg))
            kids = [int(x) for x in rng.integers(0, vocab, 20)] + [ref, ref]  # duplicates: first one wins
            tok, child = match(lg, kids)
            assert tok == ref, (vocab, dtype)
            assert child == kids.index(ref)
            assert match(lg, [t for t in kids if t != ref])[1] == -1
    lg = rng.standard_normal(5000).astype(np.float32)
    lg[123] = np.nan
    lg[77] = np.nan
    assert match(lg, [3, 77])[0] == int(np.argmax(lg)) == 77
    many = [int(x) for x in rng.permutation(5000)[:2000]]  # > 1024 children: the strided match loop
    lg = rng.standard_normal(5000).astype(np.float32)
    assert match(lg, many) == (int(np.argmax(lg)), many.index(int(np.argmax(lg))) if int(np.argmax(lg)) in many else -1)
    rows = rng.standard_normal((9, 32000)).astype(np.float32)
    rows[4, 10] = rows[4, 20] = rows[4].max() + 2
    t = torch.from_numpy(rows).cuda()
    out = np.zeros(9, dtype=np.int32)
    _lib.check(lib.tp_debug_argmax(0, C.c_void_p(t.data_ptr()), 0, 32000, 9, None, 0, out.ctypes.data))
    assert out.tolist() == [int(np.argmax(r)) for r in rows]


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 4, 16, 32])
def test_topk_rows_vs_torch(k):
    """The draft model's top-k kernel: ids of the k largest logits per row, value
    descending, lowest id first on ties (checked on rows with planted ties)."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(k)
    logits = torch.randn(37, 32000, device="cuda", generator=g)
    logits[3, 100] = logits[3, 7] = 50.0  # a tie at the top: id 7 first
    m = tp.LlamaModel(tp.LlamaConfig(vocab=512, hidden=256, layers=1, heads=2, kv_heads=1, ffn=512), max_nodes=16)
    got = m.topk_many(logits, k).cpu()
    want = torch.topk(logits, k, dim=1)
    assert torch.equal(torch.gather(logits.cpu(), 1, got.long()), want.values.cpu())
    assert int(got[3, 0]) == 7 and (k == 1 or int(got[3, 1]) == 100)
    vals = torch.gather(logits.cpu(), 1, got.long())
    assert bool((vals[:, :-1] >= vals[:, 1:]).all())
