"""GPU parity of the toy-arch path (float64 kernels) against the oracle and the
reference fixtures.  Everything here calls through libtreepipe_b200.so."""

import numpy as np
import pytest
import torch

from conftest import PIPE_CASES, ListReplay, golden_npz, pipeline_case
from oracle.lcg import uniform_stream
from oracle.pipeline import OracleRunner
from oracle.toy import OracleKv, ToyOracle, forward_nodes, greedy_continuation

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200.model import KvCache, forward_tree, kv_prune  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineRunner  # noqa: E402

TOL = 1e-12  # float64 kernels vs the float64 reference (different summation order)


def close(a, b, tol=TOL):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(1.0, float(np.max(np.abs(b)))) if b.size else 1.0
    err = float(np.max(np.abs(a - b))) if b.size else 0.0
    assert err <= tol * scale, err


def test_device_lcg_bit_exact():
    g = golden_npz("lcg.npz")
    for seed in (0, 11, 123456789):
        assert np.array_equal(tp.lcg_uniform_stream(seed, 256), g[f"seed{seed}"])
    assert np.array_equal(tp.lcg_uniform_stream(7, 5000, start=12345), uniform_stream(7, 5000, start=12345))


def test_weights_bit_exact():
    cfg = tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=11)
    m = tp.init_model(cfg)
    o = ToyOracle(32, 8, 2, 11)
    assert np.array_equal(m.embedding, o.embedding)
    for layer in range(2):
        w = m.layer_weights(layer)
        for k in ("wq", "wk", "wv", "wo", "w1", "w2"):
            assert np.array_equal(w[k], o.blocks[layer][k])


def test_forward_tree_vs_reference_fixture(golden):
    g = golden_npz("toy_model.npz")
    m = tp.init_model(tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=11))
    cache = KvCache(2, 8)
    for pos, tok in enumerate([3, 11, 4]):
        m.forward_position(m.embed(tok, pos), cache, list(range(len(cache))), uid=-1, position=pos, prefix=True)
    nodes = [(100, 5, 3, frozenset({100})), (101, 9, 3, frozenset({101})), (102, 1, 4, frozenset({100, 102})),
             (103, 2, 4, frozenset({100, 103})), (104, 7, 4, frozenset({101, 104})),
             (105, 30, 5, frozenset({100, 102, 105}))]
    out = forward_tree(m, cache, nodes)
    close(out, g["tree_out"])
    for layer in range(2):
        close(cache.keys[layer], g[f"tree_k{layer}"])
        close(cache.values[layer], g[f"tree_v{layer}"])
    close(m.head(out[-1]), g["head"])
    close(m.embed(5, 3), g["embed_5_3"])
    for prompt, want in golden["sequential"].items():
        assert tp.sequential_decode(m, eval(prompt), 24) == want


@pytest.mark.parametrize("idx", PIPE_CASES)
def test_pipeline_matches_reference_dump(golden, idx):
    """Tokens, hit/miss, KV keep lists and tree bytes bit-exact; stage outputs ≤1e-12."""
    case = pipeline_case(golden, idx)
    mc = case["model"]
    model = tp.init_model(tp.ToyModelConfig(**mc))
    runner = PipelineRunner(model, tp.PipelineConfig(num_stages=case["stages"]),
                            tp.BeamConfig(w=case["w"], k=case["k"]), ListReplay(case["trace"]))
    runner.prefill(case["prompt"])
    arrays = golden_npz(f"pipe_{case['name']}.npz")
    captured = {}
    orig = runner.launch_compute

    def spy():
        fresh = not runner._computed
        orig()
        if fresh:
            for stage in runner.stages:
                captured[stage.stage_id - 1] = None if stage.out is None else stage.out.detach().cpu().numpy()

    runner.launch_compute = spy
    for si, want in enumerate(case["steps"]):
        captured.clear()
        o = runner.decode_step()
        assert o.verified_token == want["token"], si
        assert o.hit == want["hit"], si
        assert o.flush_depth == want["flush_depth"], si
        assert runner.last_keeps == want["keeps"], si
        assert tp.encode(runner.tree).hex() == want["tree"], si
        for j in range(case["stages"]):
            key = f"s{si}_stage{j}"
            if key in arrays:
                close(captured[j], arrays[key])
    assert runner.emitted == case["emitted"]


def test_losslessness_random_triples():
    """Acceptance-1 analogue: SpecPipe on GPU == CPU oracle greedy decode (and
    == GPU sequential decode) over random model/prompt/draft triples."""
    rng = np.random.default_rng(2024)
    for model_seed in range(6):
        cfg = tp.ToyModelConfig(vocab=64, hidden=32, layers=8, seed=model_seed)
        model = tp.init_model(cfg)
        oracle = ToyOracle(64, 32, 8, model_seed)
        for j in range(3):
            prompt = [int(t) for t in rng.integers(0, 64, size=int(rng.integers(1, 5)))]
            miss = [0.0, 0.05, 0.5, 1.0][(model_seed + j) % 4]
            draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=min(0.7, 1 - miss), rank_decay=0.5,
                                                              miss_prob=miss, seed=int(rng.integers(1 << 30))), 64)
            stages = int(rng.choice([2, 4]))
            want = greedy_continuation(oracle, prompt, 48)
            res = tp.run(model, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=2, k=2), draft, prompt, 48,
                         collect_trace=False)
            assert res.tokens == want, (model_seed, prompt, miss)


def test_batch_invariance_bitwise():
    """A node's output bits do not depend on its launch-mates (sibling isolation,
    reference test_model.py:127-139, strengthened to batch composition)."""
    cfg = tp.ToyModelConfig(vocab=32, hidden=16, layers=2, seed=4)
    m = tp.init_model(cfg)

    def fresh():
        c = KvCache(2, 16)
        for pos, tok in enumerate([3, 7, 1]):
            m.forward_position(m.embed(tok, pos), c, list(range(len(c))), uid=-1, position=pos, prefix=True)
        return c

    nodes = [(10 + i, (5 * i) % 32, 3, frozenset({10 + i})) for i in range(9)]
    together = forward_tree(m, fresh(), nodes).cpu().numpy()
    for i, nd in enumerate(nodes):
        alone = forward_tree(m, fresh(), [nd]).cpu().numpy()
        assert np.array_equal(alone[0], together[i])
    rev = forward_tree(m, fresh(), nodes[::-1]).cpu().numpy()
    assert np.array_equal(rev[::-1], together)


def _random_tree(rng, vocab, max_nodes):
    t = tp.new_root(int(rng.integers(vocab)), vocab)
    while t.size < max_nodes:
        lo, hi = t.level_bounds(t.num_levels - 1)
        ch = []
        for p in range(lo, hi):
            for prob in sorted(rng.random(int(rng.integers(0, 4))), reverse=True):
                ch.append((p, int(rng.integers(vocab)), float(prob)))
        ch = ch[: max_nodes - t.size]
        if not ch or rng.random() < 0.1:
            break
        t = tp.layer_append(t, ch)
    return t


def test_tree_mask_forward_vs_oracle():
    """Acceptance-2 analogue: whole-tree forward on GPU vs the oracle (≤1e-9)."""
    cfg = tp.ToyModelConfig(vocab=16, hidden=8, layers=2, seed=1)
    m = tp.init_model(cfg)
    o = ToyOracle(16, 8, 2, 1)
    rng = np.random.default_rng(7)
    prompt = [3, 11]
    for case in range(20):
        t = _random_tree(rng, 16, int(rng.choice([8, 32, 64, 200])))
        cache, okv = KvCache(2, 8), OracleKv(2, 8)
        for pos, tok in enumerate(prompt):
            m.forward_position(m.embed(tok, pos), cache, list(range(len(cache))), uid=-1, position=pos, prefix=True)
            o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
        nodes = [(100 + i, int(t.tokens[i]), 2 + t.depth_of(i),
                  frozenset(100 + int(j) for j in np.flatnonzero(t.mask[i])[:-1])) for i in range(t.size)]
        got = forward_tree(m, cache, nodes).cpu().numpy()
        want = forward_nodes(o, okv, nodes)
        assert np.max(np.abs(got - want)) <= 1e-9


def test_kv_prune_vs_oracle():
    """Acceptance-3 analogue: chained reroot prunes keep exactly the oracle's rows."""
    cfg = tp.ToyModelConfig(vocab=16, hidden=8, layers=2, seed=2)
    m = tp.init_model(cfg)
    o = ToyOracle(16, 8, 2, 2)
    rng = np.random.default_rng(11)
    prompt = [5, 1, 9]
    for case in range(10):
        t = _random_tree(rng, 16, 40)
        cache, okv = KvCache(2, 8), OracleKv(2, 8)
        for pos, tok in enumerate(prompt):
            m.forward_position(m.embed(tok, pos), cache, list(range(len(cache))), uid=-1, position=pos, prefix=True)
            o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
        nodes = [(t.uids[i], int(t.tokens[i]), 3 + t.depth_of(i),
                  frozenset(t.uids[int(j)] for j in np.flatnonzero(t.mask[i])[:-1])) for i in range(t.size)]
        forward_tree(m, cache, nodes)
        forward_nodes(o, okv, nodes)
        cur, chains = t, set()
        for _ in range(int(rng.integers(1, 3))):
            if cur.size == 1:
                break
            target = int(rng.integers(1, cur.size))
            chains |= {cur.uids[int(j)] for j in tp.mask_row(cur, target).indices()}
            cur, _ = tp.to_subtree_prune(cur, target)
            keep = set(cur.uids) | chains
            kv_prune(cache, keep)
            okv.restrict(okv.keep_rows(keep))
        assert cache.uids == okv.uids
        assert cache.prefix_flags[:3] == [True] * 3
        for layer in range(2):
            close(cache.keys[layer], okv.keys(layer))
            close(cache.values[layer], okv.values(layer))


def test_worker_mode_bit_identical():
    cfg = tp.ToyModelConfig(vocab=48, hidden=8, layers=4, seed=9)
    m = tp.init_model(cfg)

    def one(execution):
        d = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1, seed=77), 48)
        r = tp.run(m, tp.PipelineConfig(num_stages=3, execution=execution), tp.BeamConfig(w=3, k=3), d, [2, 4], 32)
        return r.tokens, r.metrics.to_json(), r.trace

    assert one("single") == one("single") == one("workers")


def test_vanilla_and_brackets():
    cfg = tp.ToyModelConfig(vocab=48, hidden=16, layers=8, seed=4)
    m = tp.init_model(cfg)
    want = greedy_continuation(ToyOracle(48, 16, 8, 4), [1, 2], 24)
    for stages in (2, 4, 8):
        van = tp.run_vanilla(m, tp.PipelineConfig(num_stages=stages), [1, 2], 24, collect_trace=False)
        assert van.tokens == want and van.metrics.steps_per_token == float(stages)
        perfect = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=1.0, miss_prob=0.0), 48)
        r = tp.run(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=2, k=2), perfect, [1, 2], 24,
                   collect_trace=False)
        assert r.tokens == want and r.metrics.steps_per_token == 1.0
        hopeless = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.0, rank_decay=0.0, miss_prob=1.0), 48)
        r = tp.run(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=2, k=2), hopeless, [1, 2], 24,
                   collect_trace=False)
        assert r.tokens == want and r.metrics.steps_per_token == float(stages)
