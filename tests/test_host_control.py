"""Host-control mirror (tree / draft / expansion / perf) vs reference fixtures."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2504_04104_b200 as tp
from paper_2504_04104_b200.errors import InvalidTokenError, OrderingError, TreeStructureError
from paper_2504_04104_b200.tree import pack_rows, unpack_rows


def build(root, levels, vocab=32):
    t = tp.new_root(root, vocab)
    for lv in levels:
        t = tp.layer_append(t, [tuple(c) for c in lv])
    return t


def test_trees_bit_exact(golden):
    for case in golden["trees"]:
        t = build(case["root"], case["levels"])
        assert tp.encode(t).hex() == case["encoded"]
        pruned, surv = tp.to_subtree_prune(t, case["reroot"])
        assert tp.encode(pruned).hex() == case["pruned"]
        assert surv.indices().tolist() == case["survivors"]
        assert [tp.cumulative_prob(t, j) for j in range(t.size)] == case["cum"]
        back = tp.decode(bytes.fromhex(case["encoded"]), vocab_size=32)
        assert tp.structurally_equal(back, t)
        tp.validate(t)
        tp.validate(pruned)


def test_expand_bit_exact(golden):
    class Table:
        def __init__(self, table):
            self.table = {int(k): [tuple(c) for c in v] for k, v in table.items()}

        def propose(self, context, k, *, step=0, frontier_node=0):
            return self.table[frontier_node][:k]

    for case in golden["expand"]:
        t = build(0, case["levels"], vocab=64)
        got = tp.expand_fixed_width(t, tp.BeamConfig(w=case["w"], k=case["k"]), Table(case["table"]), (0,))
        assert [list(c) for c in got] == case["expected"]


def test_synthetic_draft_bit_exact(golden):
    for c in golden["draft"]:
        cfg = tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=c["seed"])
        got = tp.synthetic_draft(cfg, c["next"], c["k"], c["call"], 64)
        assert [[t, p] for t, p in got] == c["out"]


def test_perf_matches(golden):
    g = golden["perf"]
    for p, m, spt, hits, misses in g["cadence"]:
        s = tp.simulate_cadence(p, m, tokens=2000, seed=1234 + m)
        assert (s.steps_per_token, s.hits, s.misses) == (spt, hits, misses)
    cost = tp.CostModel(base_ms=40, slope_ms_per_quantum=8, quantum=64)
    widths = (1, 2, 4, 8, 16, 32, 64, 128)
    curve = tp.AccuracyCurve(widths, (0.55, 0.68, 0.80, 0.88, 0.93, 0.96, 0.99, 0.992))
    assert tp.select_width(cost, curve, 4, widths) == g["select"]
    assert [tp.step_cost(cost, w) for w in (1, 63, 64, 65, 128, 129)] == g["steps"]


def test_append_errors():
    t = tp.new_root(0, 32)
    with pytest.raises(InvalidTokenError):
        tp.new_root(32, 32)
    with pytest.raises(OrderingError):
        tp.layer_append(t, [(0, 1, 0.2), (0, 2, 0.9)])
    t2 = tp.layer_append(t, [(0, 1, 0.5)])
    with pytest.raises(TreeStructureError):
        tp.layer_append(t2, [(0, 2, 0.5)])
    with pytest.raises(InvalidTokenError):
        tp.layer_append(t, [(0, 99, 0.5)])
    with pytest.raises(TreeStructureError):
        tp.layer_append(t, [])


def _random_tree(seed, max_nodes=300):
    rng = np.random.default_rng(seed)
    t = tp.new_root(int(rng.integers(32)), 32)
    while t.size < max_nodes and rng.random() < 0.9:
        lo, hi = t.level_bounds(t.num_levels - 1)
        ch = []
        for p in range(lo, hi):
            for prob in sorted(rng.random(int(rng.integers(0, 4))), reverse=True):
                ch.append((p, int(rng.integers(32)), float(prob)))
        ch = ch[: max_nodes - t.size]
        if not ch:
            break
        t = tp.layer_append(t, ch)
    return t


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 2**31 - 1))
def test_bits_match_parent_pointers_and_roundtrip(seed):
    t = _random_tree(seed)
    n = t.size
    want = np.zeros((n, n), bool)
    for i in range(n):
        j = i
        want[i, i] = True
        while (p := t.parent_of(j)) is not None:
            want[i, p] = True
            j = p
    assert np.array_equal(t.mask, want)
    assert np.array_equal(unpack_rows(pack_rows(want), n), want)
    r = int(np.random.default_rng(seed).integers(n))
    pruned, surv = tp.to_subtree_prune(t, r)
    tp.validate(pruned)
    assert np.array_equal(pruned.mask, t.mask[np.ix_(surv.indices(), surv.indices())])


def test_native_synthetic_draft_bit_exact():
    """The native restatement of numpy's SeedSequence/PCG64/choice draws equals
    synthetic_draft (itself pinned to the reference by the golden fixtures)."""
    import ctypes as C

    from paper_2504_04104_b200 import _lib
    from paper_2504_04104_b200.token_source import SyntheticDraftConfig, synthetic_draft

    lib = _lib.load()
    rng = np.random.default_rng(99)
    checked = 0
    for _ in range(3000):
        V = int(rng.choice([16, 64, 512, 32000]))
        k = int(rng.integers(1, min(V - 1, 33)))
        miss = float(rng.choice([0.0, 0.01, 0.2]))
        cfg = SyntheticDraftConfig(top1_hit=min(float(rng.choice([0.0, 0.62, 1.0])), 1 - miss),
                                   rank_decay=float(rng.choice([0.0, 0.5, 0.6])), miss_prob=miss,
                                   seed=int(rng.choice([0, 3, 2**35 + 1])))
        idx = int(rng.integers(0, 1 << 30))
        nxt = None if rng.random() < 0.2 else int(rng.integers(0, V))
        want = [t for t, _ in synthetic_draft(cfg, nxt, k, idx, V)]
        out = np.zeros(k, np.int32)
        n = C.c_int32()
        rc = lib.tp_synthetic_draft(cfg.seed, idx, -1 if nxt is None else nxt, cfg.top1_hit, cfg.rank_decay,
                                    cfg.miss_prob, k, V, out.ctypes.data, C.byref(n))
        assert rc == 0
        assert out[: n.value].tolist() == want
        checked += 1
    assert checked == 3000


@pytest.mark.parametrize("w,k,levels", [(64, 16, 6), (8, 4, 4), (3, 3, 7), (1, 2, 5)])
def test_batched_expand_equals_per_node(w, k, levels):
    """expand_fixed_width's native batched path == the per-node reference loop."""
    V = 32000
    truth = tuple(int(t) for t in np.random.default_rng(w * 7 + k).integers(0, V, 900))
    ctx = truth[:300]
    fast_d = tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=4), V)
    slow_d = tp.RecordingDraft(tp.SyntheticDraft(tp.SyntheticDraftConfig(seed=4), V))  # no propose_batch
    fast_d.bind_reference(truth)
    slow_d.bind_reference(truth)
    beam = tp.BeamConfig(w=w, k=k)
    tree = tp.new_root(ctx[-1], V)
    for _ in range(levels):
        a = tp.expand_fixed_width(tree, beam, fast_d, ctx)
        b = tp.expand_fixed_width(tree, beam, slow_d, ctx)
        assert a == b
        tree = tp.layer_append(tree, a)
    assert fast_d._calls == slow_d.inner._calls


def test_draft_model_shapes():
    """The draft-model configs the bench runs (BASELINE configs 2 and 4): the 68M
    shape with the kernels' 128-wide heads keeps JackFram/llama-68m's parameter
    count; the 7B draft of config 4 is the 7B target shape with its own seed."""
    from paper_2504_04104_b200.model import LlamaConfig

    c = LlamaConfig.llama_68m()
    assert (c.hidden, c.layers, c.ffn, c.vocab, c.heads * c.head_dim) == (768, 2, 3072, 32000, 768)
    assert abs(c.param_count - 68.0e6) < 0.5e6
    assert c.seed != LlamaConfig.llama2_7b().seed
