"""Generate golden fixtures from the UNMODIFIED reference (build container only).

Run:  python tests/golden/make_golden.py   (needs /root/reference; the GPU box
never runs this — it only reads the committed fixtures).

Everything recorded here comes from calling the reference's public API
(`/root/reference/pkg/src/treepipe`).  Per-step KV keep lists are captured
by wrapping ``KvCache._restrict`` (`model.py:184`), the only place the
reference compacts a cache.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import treepipe as tp  # noqa: E402
from treepipe import model as tp_model  # noqa: E402
from treepipe.pipeline import PipelineRunner  # noqa: E402


def lcg_fixture():
    out = {}
    for seed in (0, 11, 123456789):
        out[f"seed{seed}"] = tp.lcg_uniform_stream(seed, 256)
    return out


def random_tree(rng, vocab, max_nodes):
    tree = tp.new_root(int(rng.integers(vocab)), vocab)
    steps = [int(tree.tokens[0])]
    levels = []
    while tree.size < max_nodes:
        lo, hi = tree.level_bounds(tree.num_levels - 1)
        children = []
        for parent in range(lo, hi):
            for prob in sorted(rng.random(int(rng.integers(0, 4))), reverse=True):
                children.append((parent, int(rng.integers(vocab)), float(prob)))
        children = children[: max_nodes - tree.size]
        if not children or rng.random() < 0.1:
            break
        tree = tp.layer_append(tree, children)
        levels.append(children)
    return tree, steps[0], levels


def tree_fixture():
    rng = np.random.default_rng(5)
    cases = []
    for i in range(40):
        tree, root, levels = random_tree(rng, 32, int(rng.choice([8, 40, 100, 200])))
        r = int(rng.integers(tree.size))
        pruned, surv = tp.to_subtree_prune(tree, r)
        cases.append({
            "root": root, "levels": [[list(c) for c in lv] for lv in levels],
            "encoded": tp.encode(tree).hex(), "reroot": r,
            "pruned": tp.encode(pruned).hex(), "survivors": surv.indices().tolist(),
            "cum": [tp.cumulative_prob(tree, j) for j in range(tree.size)],
        })
    return cases


class Table:
    def __init__(self, table):
        self.table = table

    def propose(self, context, k, *, step=0, frontier_node=0):
        return self.table[frontier_node][:k]


def expand_fixture():
    rng = np.random.default_rng(21)
    cases = []
    for _ in range(60):
        tree = tp.new_root(0, 64)
        levels = []
        for _ in range(int(rng.integers(1, 3))):
            lo, hi = tree.level_bounds(tree.num_levels - 1)
            ch = []
            for parent in range(lo, hi):
                for prob in sorted(rng.random(int(rng.integers(1, 3))), reverse=True):
                    ch.append((parent, int(rng.integers(64)), float(prob)))
            ch = ch[:6]
            tree = tp.layer_append(tree, ch)
            levels.append([list(c) for c in ch])
        k, w = int(rng.integers(2, 6)), int(rng.integers(1, 9))
        lo, hi = tree.level_bounds(tree.num_levels - 1)
        table = {node: [(int(t), float(p)) for t, p in zip(rng.choice(64, size=k, replace=False),
                                                            np.sort(rng.random(k))[::-1])]
                 for node in range(lo, hi)}
        got = tp.expand_fixed_width(tree, tp.BeamConfig(w=w, k=k), Table(table), (0,))
        cases.append({"levels": levels, "k": k, "w": w,
                      "table": {str(n): [list(c) for c in v] for n, v in table.items()},
                      "expected": [list(c) for c in got]})
    return cases


def draft_fixture():
    cases = []
    for seed in (0, 5, 77):
        cfg = tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=seed)
        for call in range(30):
            for nxt in (None, 3):
                for k in (2, 4, 16):
                    got = tp.synthetic_draft(cfg, nxt, k, call, 64)
                    cases.append({"seed": seed, "call": call, "next": nxt, "k": k,
                                  "out": [[int(t), float(p)] for t, p in got]})
    return cases


def perf_fixture():
    out = {"cadence": [], "select": None}
    for p in (0.8, 0.95):
        for m in (4, 8):
            s = tp.simulate_cadence(p, m, tokens=2000, seed=1234 + m)
            out["cadence"].append([p, m, s.steps_per_token, s.hits, s.misses])
    cost = tp.CostModel(base_ms=40, slope_ms_per_quantum=8, quantum=64)
    widths = (1, 2, 4, 8, 16, 32, 64, 128)
    curve = tp.AccuracyCurve(widths, (0.55, 0.68, 0.80, 0.88, 0.93, 0.96, 0.99, 0.992))
    out["select"] = tp.select_width(cost, curve, 4, widths)
    out["steps"] = [tp.step_cost(cost, w) for w in (1, 63, 64, 65, 128, 129)]
    return out


def model_fixture():
    model = tp.init_model(tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=11))
    arrays = {}
    seqs = {}
    for prompt in ([1, 2], [5, 9, 3], [7]):
        seqs[str(prompt)] = tp.sequential_decode(model, prompt, 24)
    # a small tree forwarded over a 3-token prefix, recorded fully
    cache = tp.KvCache(2, 8)
    for pos, tok in enumerate([3, 11, 4]):
        model.forward_position(model.embed(tok, pos), cache, list(range(len(cache))),
                               uid=-1, position=pos, prefix=True)
    nodes = [(100, 5, 3, frozenset({100})), (101, 9, 3, frozenset({101})),
             (102, 1, 4, frozenset({100, 102})), (103, 2, 4, frozenset({100, 103})),
             (104, 7, 4, frozenset({101, 104})), (105, 30, 5, frozenset({100, 102, 105}))]
    outs = tp.forward_tree(model, cache, nodes)
    arrays["tree_out"] = outs
    for layer in range(2):
        arrays[f"tree_k{layer}"] = cache.keys[layer]
        arrays[f"tree_v{layer}"] = cache.values[layer]
    arrays["head"] = model.head(outs[-1])
    arrays["embed_5_3"] = model.embed(5, 3)
    return seqs, arrays


def pipeline_case(name, mcfg, stages, w, k, dcfg, prompt, tokens, keep_outs_steps):
    model = tp.init_model(tp.ToyModelConfig(**mcfg))
    reference = tp.sequential_decode(model, prompt, tokens)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(**dcfg), mcfg["vocab"])
    rec = tp.RecordingDraft(draft)
    rec.bind_reference(tuple(prompt) + tuple(reference))
    runner = PipelineRunner(model, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=w, k=k),
                            rec, collect_trace=False)
    restricts = []
    orig = tp_model.KvCache._restrict

    def spy(self, keep):
        restricts.append((id(self), list(keep)))
        return orig(self, keep)

    tp_model.KvCache._restrict = spy
    try:
        runner.prefill(prompt)
        kv_ids = [id(s.kv) for s in runner.stages]
        steps, arrays = [], {}
        while len(runner.emitted) < tokens:
            restricts.clear()
            outs = {}
            orig_forward = tp.pipeline.forward_tree

            def fwd(*a, **kw):
                res = orig_forward(*a, **kw)
                outs[id(a[1])] = res
                return res

            tp.pipeline.forward_tree = fwd
            try:
                o = runner.decode_step()
            finally:
                tp.pipeline.forward_tree = orig_forward
            keeps = None
            if restricts:
                keeps = [next(kk for kid, kk in restricts if kid == sid) for sid in kv_ids]
            si = len(steps)
            if si < keep_outs_steps:
                for j, sid in enumerate(kv_ids):
                    if sid in outs:
                        arrays[f"s{si}_stage{j}"] = outs[sid]
            steps.append({"token": o.verified_token, "hit": o.hit, "stalled": o.stalled,
                          "flush_depth": o.flush_depth, "keeps": keeps,
                          "tree": tp.encode(runner.tree).hex(),
                          "resident": [None if s.resident is None else len(s.resident)
                                       for s in runner.stages]})
    finally:
        tp_model.KvCache._restrict = orig
    m = runner.metrics()
    meta = {"name": name, "model": mcfg, "stages": stages, "w": w, "k": k, "draft": dcfg,
            "prompt": prompt, "tokens": tokens, "reference": reference, "emitted": runner.emitted,
            "steps": steps, "metrics": m.to_json(), "trace": rec.records}
    return meta, arrays


def main():
    np.savez_compressed(os.path.join(HERE, "lcg.npz"), **lcg_fixture())
    seqs, arrays = model_fixture()
    np.savez_compressed(os.path.join(HERE, "toy_model.npz"), **arrays)
    cases = [
        ("tiny_m3", dict(vocab=48, hidden=8, layers=4, seed=3), 3, 3, 3,
         dict(top1_hit=0.7, rank_decay=0.5, miss_prob=0.1, seed=9), [2, 4], 24, 1000),
        ("tiny_m4_miss", dict(vocab=48, hidden=16, layers=8, seed=4), 4, 2, 2,
         dict(top1_hit=0.5, rank_decay=0.5, miss_prob=0.3, seed=2), [1, 2, 3], 20, 1000),
        ("c1_cli", dict(vocab=64, hidden=256, layers=4, seed=0), 2, 4, 4,
         dict(top1_hit=0.62, rank_decay=0.6, miss_prob=0.01, seed=0), list(range(1, 17)), 24, 6),
    ]
    pipes = []
    for case in cases:
        meta, arr = pipeline_case(*case)
        pipes.append(meta)
        np.savez_compressed(os.path.join(HERE, f"pipe_{meta['name']}.npz"), **arr)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump({"sequential": seqs, "trees": tree_fixture(), "expand": expand_fixture(),
                   "draft": draft_fixture(), "perf": perf_fixture(), "pipelines": pipes}, fh)
    c1_paper()
    artefacts()


def artefacts():
    """Reference-written on-disk artefacts: the checkpoint file
    (`model.py:388-435`), the StepTrace CSV (`pipeline.py:123-152`) and the
    RunMetrics JSON of a replayed run, plus the draft-trace JSONL
    (`token_source.py:178-226`)."""
    import io

    model = tp.init_model(tp.ToyModelConfig(vocab=32, hidden=8, layers=2, seed=11))
    tp_model.save_checkpoint(model, os.path.join(HERE, "ref_ckpt_v32_d8_l2_s11.bin"))
    cfg = dict(vocab=48, hidden=8, layers=4, seed=3)
    model = tp.init_model(tp.ToyModelConfig(**cfg))
    prompt = [2, 4]
    reference = tp.sequential_decode(model, prompt, 24)
    rec = tp.RecordingDraft(tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5,
                                                                       miss_prob=0.1, seed=9), 48))
    rec.bind_reference(tuple(prompt) + tuple(reference))
    res = tp.run(model, tp.PipelineConfig(num_stages=3), tp.BeamConfig(w=3, k=3), rec, prompt, 24)
    buf = io.StringIO()
    tp.write_trace_csv(res.trace, buf)
    with open(os.path.join(HERE, "ref_trace_m3.csv"), "w", newline="") as fh:
        fh.write(buf.getvalue())
    with open(os.path.join(HERE, "ref_metrics_m3.json"), "w") as fh:
        json.dump({"model": cfg, "prompt": prompt, "stages": 3, "w": 3, "k": 3, "tokens": res.tokens,
                   "metrics": res.metrics.to_json()}, fh)
    tp.write_trace(rec.records, os.path.join(HERE, "ref_draft_m3.jsonl"))


def c1_paper():
    """C1 with the paper beam: ToyModel V=64, d=256, L=4, 2 stages,
    w=64 / k=16, a 128-token prompt, the paper-calibrated synthetic draft."""
    prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, 64, 128)]
    meta, arr = pipeline_case("c1_paper", dict(vocab=64, hidden=256, layers=4, seed=0), 2, 64, 16,
                              dict(top1_hit=0.62, rank_decay=0.6, miss_prob=0.01, seed=0), prompt, 32, 4)
    np.savez_compressed(os.path.join(HERE, "pipe_c1_paper.npz"), **arr)
    with open(os.path.join(HERE, "pipe_c1_paper.json"), "w") as fh:
        json.dump(meta, fh)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if "c1_paper" in sys.argv:
        c1_paper()
    elif "artefacts" in sys.argv:
        artefacts()
    else:
        main()
