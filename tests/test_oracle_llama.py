"""Self-validation of the Llama oracle (oracle/llama.py) with the reference's
own acceptance logic, restated for the Llama arch (CPU only):

* acceptance 2 (`/root/reference/pkg/tests/test_acceptance.py:82-143`): every
  leaf's tree-forward output equals a from-scratch causal forward along its
  root path — here bit for bit, since both issue the same float32 ops;
* acceptance 3 (`test_acceptance.py:146-212`): after chained reroot prunes
  with the row-or-column keep rule, the kept K/V rows equal a from-scratch
  recompute and the verified prefix is never dropped;
* the batched restatements used at the benchmark shapes (``prefill_block``,
  ``forward_level``) agree with the per-node ones within float32 rounding.
"""

import numpy as np

from oracle.llama import LlamaOracle
from oracle.toy import forward_nodes
from paper_2504_04104_b200 import tree as T

SHAPE = dict(vocab=64, hidden=256, layers=2, heads=2, kv_heads=1, ffn=384)


def random_tree(rng, vocab, max_nodes):
    tree = T.new_root(int(rng.integers(vocab)), vocab)
    while tree.size < max_nodes:
        lo, hi = tree.level_bounds(tree.num_levels - 1)
        children = []
        for parent in range(lo, hi):
            for prob in sorted(rng.random(int(rng.integers(0, 4))), reverse=True):
                children.append((parent, int(rng.integers(vocab)), float(prob)))
        children = children[: max_nodes - tree.size]
        if not children:
            break
        tree = T.layer_append(tree, children)
    return tree


def ancestors(tree, i, uid_of):
    return frozenset(uid_of(int(j)) for j in T.mask_row(tree, i).indices()[:-1])


def prefix(o, prompt, dense=False):
    kv = o.new_dense_kv() if dense else o.new_kv()
    x = None
    for pos, tok in enumerate(prompt):
        x = o.run_position(o.embed(tok, pos), kv, list(range(len(kv))), pos=pos, prefix=True)
    return kv, x


def test_acceptance2_tree_forward_equals_path_forward():
    o = LlamaOracle(**SHAPE)
    rng = np.random.default_rng(7)
    prompt = [3, 11, 40]
    checked = 0
    for _ in range(6):
        tree = random_tree(rng, SHAPE["vocab"], int(rng.choice([8, 16, 30])))
        kv, _ = prefix(o, prompt)
        base = len(prompt)
        nodes = [(100 + i, int(tree.tokens[i]), base + tree.depth_of(i), ancestors(tree, i, lambda j: 100 + j))
                 for i in range(tree.size)]
        outs = forward_nodes(o, kv, nodes)
        parents = {tree.parent_of(i) for i in range(tree.size)}
        for leaf in (i for i in range(tree.size) if i not in parents):
            path = [int(j) for j in T.mask_row(tree, leaf).indices()]
            _, x = prefix(o, prompt + [int(tree.tokens[j]) for j in path])
            assert np.array_equal(outs[leaf], x), leaf
            checked += 1
    assert checked > 10


def test_acceptance3_pruned_kv_equals_recompute():
    o = LlamaOracle(**SHAPE)
    rng = np.random.default_rng(11)
    prompt = [5, 1, 9]
    base = len(prompt)
    for _ in range(6):
        tree = random_tree(rng, SHAPE["vocab"], 30)
        kv, _ = prefix(o, prompt)
        node = lambda t, i: (t.uids[i], int(t.tokens[i]), base + t.depth_of(i),  # noqa: E731
                             ancestors(t, i, lambda j: t.uids[j]))
        forward_nodes(o, kv, [node(tree, i) for i in range(tree.size)])
        current, chains = tree, set()
        for _ in range(int(rng.integers(1, 3))):
            if current.size == 1:
                break
            target = int(rng.integers(1, current.size))
            chains |= {current.uids[int(j)] for j in T.mask_row(current, target).indices()}
            current, _ = T.to_subtree_prune(current, target)
            kv.restrict(kv.keep_rows(set(current.uids.tolist() if hasattr(current.uids, "tolist")
                                         else current.uids) | chains))
        assert [i for i, p in enumerate(kv.prefix) if p] == list(range(base))
        fresh, _ = prefix(o, prompt)
        kept = [u for u in kv.uids if u != -1]
        index_of = {u: i for i, u in enumerate(tree.uids)}
        for uid in kept:
            forward_nodes(o, fresh, [node(tree, index_of[uid])])
        for layer in range(SHAPE["layers"]):
            got = kv.keys(layer)[base:]
            want = fresh.keys(layer)[[fresh.uids.index(u) for u in kept]]
            assert np.array_equal(got, want)
            assert np.array_equal(kv.values(layer)[base:], fresh.values(layer)[[fresh.uids.index(u) for u in kept]])


def rel_err(got, want):
    """(max |d| / max |want|, rms(d) / rms(want)) — compared as a tuple."""
    d = np.asarray(got, np.float64) - np.asarray(want, np.float64)
    w = np.asarray(want, np.float64)
    return (float(np.abs(d).max() / max(np.abs(w).max(), 1e-30)),
            float(np.sqrt((d * d).mean()) / max(np.sqrt((w * w).mean()), 1e-30)))


def test_batched_restatement_matches_per_node():
    """prefill_block / forward_level (GEMMs over a level, masked causal
    attention) == run_position / forward_nodes up to bf16 re-rounding: the
    per-node oracle rounds h, q/k/v, P and the SwiGLU product to bf16 after
    float32 GEMVs, the batched one after float32 GEMMs; the few values whose
    float32 sums straddle a bf16 rounding boundary flip by one bf16 ulp
    (2^-8 relative), which is what the stated bound (max 2e-2, rms 5e-3 of
    the row scale) absorbs.  Tree semantics are pinned bit-exact above."""
    o = LlamaOracle(**{**SHAPE, "heads": 4, "kv_heads": 2})
    rng = np.random.default_rng(3)
    prompt = [int(t) for t in rng.integers(0, SHAPE["vocab"], 70)]
    kv_a, x_a = prefix(o, prompt)
    kv_b = o.new_dense_kv(8)
    xs = o.prefill_block(prompt, kv_b, chunk=32)
    assert all(e <= t for e, t in zip(rel_err(xs[-1], x_a), (2e-2, 5e-3)))
    for layer in range(SHAPE["layers"]):
        assert all(e <= t for e, t in zip(rel_err(kv_b.keys(layer), np.stack(kv_a.k[layer])), (2e-2, 5e-3)))
    P = len(prompt)
    lvl1 = [(10 + i, int(rng.integers(SHAPE["vocab"])), P, frozenset({10 + i})) for i in range(4)]
    lvl2 = [(20 + j, int(rng.integers(SHAPE["vocab"])), P + 1, frozenset({10 + j % 4, 20 + j})) for j in range(7)]
    for lvl in (lvl1, lvl2):
        a = forward_nodes(o, kv_a, lvl)
        b = o.forward_level(kv_b, lvl)
        assert all(e <= t for e, t in zip(rel_err(b, a), (2e-2, 5e-3)))
    assert kv_b.uids == kv_a.uids and kv_b.positions == kv_a.positions
