"""Llama parity at the BENCHMARKED shapes (BASELINE.json configs 2-4).

A real stage step is pushed through a 1-2 layer slice of the 7B (32x128 MHA),
13B (40 heads) and 70B (64/8 GQA, d=8192, f=28672) shapes, on the GPU through
the C ABI and on the CPU through the float32 oracle (oracle/llama.py, itself
validated with the reference's acceptance-2/3 logic in test_oracle_llama.py):

  prompt prefill (512 / 512 / 4096 tokens)  ->  a w=16 first tree level  ->
  a w=64 second level (4 children per node)  ->  verification hit on one
  level-1 child: promote + prune (row-or-column keep rule, pipeline.py:341-353)
  ->  a w=64 third level over the pruned cache  ->  LM-head logits.

Checked: keep lists bit-exact with the oracle's; the surviving K/V rows on the
GPU are bit-identical to the same rows before compaction; hidden outputs,
K rows and logits within the stated bf16 tolerance of the oracle; greedy
tokens equal wherever the oracle's top-1 margin exceeds the tolerance.

Tolerance (measured, see profiles/r02_llama_shape_parity.txt): the GPU and the
oracle round h, q/k/v, P and the SwiGLU product to bf16 after float32 sums
taken in different orders, so isolated values flip by one bf16 ulp (2^-8
relative).  Bound per compared tensor: max |d| <= TOL_MAX * max |oracle| and
rms(d) <= TOL_RMS * rms(oracle).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle.llama import LlamaOracle

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, forward_tree, prefill_rows  # noqa: E402

TOL_MAX = 1e-2
TOL_RMS = 2e-3

SHAPES = {
    "7b": dict(cfg=LlamaConfig.llama2_7b(), layers=(0, 2), prompt=512),
    "13b": dict(cfg=LlamaConfig.llama2_13b(), layers=(0, 2), prompt=512),
    "70b": dict(cfg=LlamaConfig.llama2_70b(), layers=(0, 1), prompt=4096),
}
LOG = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "llama_shape_parity.jsonl")


def rel_err(got, want):
    d = np.asarray(got, np.float64) - np.asarray(want, np.float64)
    w = np.asarray(want, np.float64)
    return (float(np.abs(d).max() / max(np.abs(w).max(), 1e-30)),
            float(np.sqrt((d * d).mean()) / max(np.sqrt((w * w).mean()), 1e-30)))


def as_f32(u16):
    return (np.asarray(u16).astype(np.uint32) << 16).view(np.float32)


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", list(SHAPES))
def test_stage_step_at_benchmark_shape(name):
    spec = SHAPES[name]
    cfg, (lo, hi), P = spec["cfg"], spec["layers"], spec["prompt"]
    model = LlamaModel(cfg, max_nodes=64, layer_range=(lo, hi), with_embed=True, with_head=True)
    orc = LlamaOracle(cfg.vocab, cfg.hidden, cfg.layers, cfg.heads, cfg.kv_heads, cfg.ffn, seed=cfg.seed,
                      layer_range=(lo, hi))
    rng = np.random.default_rng(100 + cfg.hidden)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, P)]
    errs = {}

    def check(tag, got, want):
        got = got.detach().float().cpu().numpy() if isinstance(got, torch.Tensor) else got
        e = rel_err(got, want)
        errs[tag] = e
        assert e[0] <= TOL_MAX and e[1] <= TOL_RMS, (tag, e)

    cache = KvCache(cfg.layers, cfg.hidden, capacity=P + 256).bind(model, (lo, hi))
    okv = orc.new_dense_kv(P + 256)
    xg = prefill_rows(model, cache, prompt, layer_range=(lo, hi))
    xo = orc.prefill_block(prompt, okv)
    check("prefill", xg[-64:], xo[-64:])

    # level 1: 16 children of the root (the last prompt token, already cached)
    w1 = [(1000 + i, int(rng.integers(cfg.vocab)), P, frozenset({1000 + i})) for i in range(16)]
    # level 2: 64 nodes, 4 per level-1 node
    w2 = [(2000 + j, int(rng.integers(cfg.vocab)), P + 1, frozenset({1000 + j // 4, 2000 + j})) for j in range(64)]
    for tag, lvl in (("level1", w1), ("level2", w2)):
        g = forward_tree(model, cache, lvl, layer_range=(lo, hi))
        o = orc.forward_level(okv, lvl)
        check(tag, g, o)
    k_before = cache.keys[lo]
    check("k_rows", as_f32(k_before[P:]), okv.keys(lo)[P:])

    # verification hit on level-1 child 5: promote the chain, prune to row-or-column
    child = 1000 + 5
    chain = {child}
    keep = chain | {1000 + 5} | {2000 + j for j in range(64) if j // 4 == 5}
    cache.promote(chain)
    cache.prune(keep)
    okv.promote(chain)
    okeep = okv.keep_rows(keep)
    okv.restrict(okeep)
    assert cache.last_keep == okeep
    assert cache.uids == okv.uids and cache.positions == okv.positions
    assert np.array_equal(cache.keys[lo], k_before[okeep])  # compaction moves rows bit for bit

    # level 3 over the pruned cache: 64 grandchildren of the 4 surviving level-2 nodes
    surv = [2000 + j for j in range(64) if j // 4 == 5]
    w3 = [(3000 + j, int(rng.integers(cfg.vocab)), P + 2, frozenset({surv[j % 4], 3000 + j})) for j in range(64)]
    g3 = forward_tree(model, cache, w3, layer_range=(lo, hi))
    o3 = orc.forward_level(okv, w3)
    check("level3_after_prune", g3, o3)

    lg = model.logits_many(g3[:8]).cpu().numpy()
    lo_ = np.stack([orc.logits(r) for r in o3[:8]])
    check("logits", lg, lo_)
    agreed = 0
    for r in range(8):
        top2 = np.sort(lo_[r])[-2:]
        if top2[1] - top2[0] > 2 * TOL_MAX * np.abs(lo_[r]).max():
            assert int(np.argmax(lg[r])) == int(np.argmax(lo_[r])), r
            agreed += 1
    os.makedirs(os.path.dirname(LOG), exist_ok=True)
    with open(LOG, "a") as fh:
        fh.write(json.dumps({"shape": name, "layers": [lo, hi], "prompt": P, "errors_max_rms": errs,
                             "argmax_checked": agreed}) + "\n")
    print(name, json.dumps(errs))
