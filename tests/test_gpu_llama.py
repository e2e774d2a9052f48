"""GPU checks of the Llama-shape bf16 path: the tcgen05 weight-streaming GEMM,
LCG weights, tree forward vs the float32 oracle (stated tolerance), batch
invariance, and SpecPipe losslessness w.r.t. the GPU greedy decode."""

import numpy as np
import pytest
import torch

from oracle.llama import LlamaOracle, bf16
from oracle.toy import forward_nodes, greedy_continuation

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200 import _lib  # noqa: E402
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, forward_tree  # noqa: E402

# bf16 path vs float32 oracle: |gpu - oracle| <= TOL * max|oracle| per output row
TOL = 2e-2  # same max bound as test_gpu_llama_shapes.py (TOL_MAX)
TINY = dict(vocab=512, hidden=256, layers=2, heads=2, kv_heads=1, ffn=512)


def gemm(w, x):
    n, k = x.shape
    out = torch.empty((n, w.shape[0]), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().tp_debug_gemm(0, w.data_ptr(), x.data_ptr(), n, w.shape[0], k, out.data_ptr(),
                                        _lib.stream_handle()))
    return out


@pytest.mark.parametrize("n_out,k", [(128, 64), (384, 256), (1024, 4096), (4096, 4096), (768, 1024)])
@pytest.mark.parametrize("n", [1, 5, 16, 33, 64])
def test_tcgen05_gemm_vs_torch(n_out, k, n):
    g = torch.Generator(device="cuda").manual_seed(n_out * 7 + k + n)
    w = (torch.randn((n_out, k), device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn((n, k), device="cuda", generator=g).to(torch.bfloat16)
    got = gemm(w, x)
    want = x.float() @ w.float().t()
    err = (got - want).abs().max().item()
    assert err <= 1e-4 * max(1.0, want.abs().max().item()), err


def test_tcgen05_gemm_batch_invariant():
    """Column results do not depend on how many node rows share the MMA (N)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    w = (torch.randn((1024, 4096), device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn((64, 4096), device="cuda", generator=g).to(torch.bfloat16)
    full = gemm(w, x)
    for n in (1, 7, 16, 17, 40):
        part = gemm(w, x[:n].contiguous())
        assert torch.equal(part, full[:n]), n


def test_tcgen05_gemm_heterogeneous_group_bitwise():
    """One grouped K2 launch over members of DIFFERENT shapes (each with its own
    stream-K plan: a draft model's layer next to a target stage's) is bit-identical
    to each member's own launch."""
    import ctypes as C

    from paper_2504_04104_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(11)
    shapes = [(12288, 4096, 3), (2304, 768, 40), (768, 3072, 17), (4096, 4096, 1)]
    ws = [(torch.randn((no, k), device="cuda", generator=g) * 0.05).to(torch.bfloat16) for no, k, _ in shapes]
    xs = [torch.randn((n, k), device="cuda", generator=g).to(torch.bfloat16) for _, k, n in shapes]
    outs = [torch.zeros((n, no), device="cuda") for no, _, n in shapes]
    cnt = len(shapes)
    arr = lambda ts: (C.c_void_p * cnt)(*[t.data_ptr() for t in ts])  # noqa: E731
    i32 = lambda v: (C.c_int32 * cnt)(*v)  # noqa: E731
    _lib.check(_lib.lib().tp_debug_gemm_hetero(0, cnt, arr(ws), arr(xs), i32([s[2] for s in shapes]),
                                               i32([s[0] for s in shapes]), i32([s[1] for s in shapes]), arr(outs),
                                               torch.cuda.current_stream().cuda_stream))
    for w, x, o in zip(ws, xs, outs):
        assert torch.equal(o, gemm(w, x))
        ref = x.float() @ w.float().t()
        assert float((o - ref).abs().max()) <= 1e-4 * float(ref.abs().max())


def tiny_model(**kw):
    cfg = LlamaConfig(**{**TINY, **kw})
    return cfg, LlamaModel(cfg, max_nodes=64), LlamaOracle(**{**TINY, **kw})


def test_llama_weights_bit_exact():
    cfg, m, o = tiny_model()
    d, q, kv, f = cfg.hidden, cfg.heads * 128, cfg.kv_heads * 128, cfg.ffn
    as_f32 = lambda u16: (u16.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    emb = as_f32(m.read_tensor(0).view(np.uint16)).reshape(cfg.vocab, d)
    assert np.array_equal(emb, o.embedding)
    for layer in range(cfg.layers):
        b = o.blocks[layer]
        qkv = as_f32(m.read_tensor(1, layer).view(np.uint16)).reshape(q + 2 * kv, d)
        assert np.array_equal(qkv[:q], b["wq"].T)
        assert np.array_equal(qkv[q:q + kv], b["wk"].T)
        assert np.array_equal(qkv[q + kv:], b["wv"].T)
        wo = as_f32(m.read_tensor(4, layer).view(np.uint16)).reshape(d, q)
        assert np.array_equal(wo, b["wo"].T)
        gu = as_f32(m.read_tensor(5, layer).view(np.uint16)).reshape(2 * f // 128, 2, 64, d)
        assert np.array_equal(gu[:, 0].reshape(f, d), b["wg"].T)
        assert np.array_equal(gu[:, 1].reshape(f, d), b["wu"].T)
        wd = as_f32(m.read_tensor(7, layer).view(np.uint16)).reshape(d, f)
        assert np.array_equal(wd, b["wd"].T)
    head = as_f32(m.read_tensor(8).view(np.uint16)).reshape(cfg.vocab, d)
    assert np.array_equal(head, o.lm_head.T)


def _prefix(m, o, prompt):
    cache, okv = KvCache(m.cfg.layers, m.cfg.hidden), o.new_kv()
    for pos, tok in enumerate(prompt):
        m.forward_position(m.embed(tok, pos), cache, list(range(len(cache))), uid=-1, position=pos, prefix=True)
        o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
    return cache, okv


def _rowwise_close(got, want, tol=TOL):
    got = got.detach().cpu().numpy() if hasattr(got, "detach") else got
    for a, b in zip(got, want):
        scale = max(1.0, float(np.abs(b).max()))
        assert float(np.abs(a - b).max()) <= tol * scale, float(np.abs(a - b).max()) / scale


def test_llama_tree_forward_vs_oracle():
    cfg, m, o = tiny_model()
    rng = np.random.default_rng(5)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, 70)]  # crosses a 64-slot chunk
    cache, okv = _prefix(m, o, prompt)
    P = len(prompt)
    # three-level tree: 3 children of the root, 2 grandchildren each
    nodes = [(100 + i, int(rng.integers(cfg.vocab)), P, frozenset({100 + i})) for i in range(3)]
    nodes += [(200 + 2 * i + j, int(rng.integers(cfg.vocab)), P + 1, frozenset({100 + i, 200 + 2 * i + j}))
              for i in range(3) for j in range(2)]
    got = forward_tree(m, cache, nodes)
    want = forward_nodes(o, okv, nodes)
    _rowwise_close(got, want)
    lg = m.logits_many(got).cpu().numpy()
    for r in range(len(nodes)):
        ol = o.logits(want[r])
        assert float(np.abs(lg[r] - ol).max()) <= TOL * max(1.0, float(np.abs(ol).max()))


def test_llama_batch_invariance_bitwise():
    cfg, m, o = tiny_model()
    rng = np.random.default_rng(9)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, 61)]

    def fresh():
        c = KvCache(cfg.layers, cfg.hidden)
        tp.model.prefill_rows(m, c, prompt)
        return c

    # level of 9 siblings at position P, then each alone
    P = len(prompt)
    nodes = [(10 + i, int(rng.integers(cfg.vocab)), P, frozenset({10 + i})) for i in range(9)]
    together = forward_tree(m, fresh(), nodes).cpu()
    for i, nd in enumerate(nodes):
        alone = forward_tree(m, fresh(), [nd]).cpu()
        assert torch.equal(alone[0], together[i]), i
    # a depth-4 chain crossing the 64-slot boundary == sequential prefill of the same tokens
    chain_toks = [int(t) for t in rng.integers(0, cfg.vocab, 5)]
    c1 = fresh()
    outs = []
    anc = set()
    for d, t in enumerate(chain_toks):
        anc = anc | {300 + d}
        outs.append(forward_tree(m, c1, [(300 + d, t, P + d, frozenset(anc))])[0].cpu())
    c2 = fresh()
    seq = tp.model.prefill_rows(m, c2, chain_toks, start_pos=P).cpu()
    for d in range(len(chain_toks)):
        assert torch.equal(outs[d], seq[d]), d


def test_llama_stage_split_bitwise():
    """Layers run as two stages (norm at the stage boundary) == one stage, bit for bit."""
    cfg, m, _ = tiny_model(layers=4)
    prompt = [int(t) for t in np.random.default_rng(2).integers(0, cfg.vocab, 77)]
    whole = KvCache(cfg.layers, cfg.hidden).bind(m, (0, 4))
    out_whole = tp.model.prefill_rows(m, whole, prompt, layer_range=(0, 4)).cpu()
    a = KvCache(cfg.layers, cfg.hidden).bind(m, (0, 1))
    b = KvCache(cfg.layers, cfg.hidden).bind(m, (1, 4))
    mid = tp.model.prefill_rows(m, a, prompt, layer_range=(0, 1))
    out_split = tp.model.prefill_rows(m, b, prompt, layer_range=(1, 4), x_in=mid).cpu()
    assert torch.equal(out_whole, out_split)


def test_llama_pipeline_lossless_and_margin_parity():
    cfg, m, o = tiny_model()
    prompt = [3, 1, 4, 1, 5, 9, 2, 6]
    n_tok = 24
    gpu_seq = tp.sequential_decode(m, prompt, n_tok)
    for stages, miss in ((2, 0.0), (2, 0.3)):
        draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=min(0.7, 1 - miss), rank_decay=0.5,
                                                          miss_prob=miss, seed=11), cfg.vocab)
        res = tp.run(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=4, k=4), draft, prompt, n_tok,
                     collect_trace=False)
        assert res.tokens == gpu_seq
    # teacher-forced agreement with the oracle wherever its top-1 margin exceeds the tolerance
    okv = o.new_kv()
    x = None
    for pos, tok in enumerate(prompt):
        x = o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
    checked = 0
    for i, tok in enumerate(gpu_seq):
        lg = o.logits(x)
        top2 = np.sort(lg)[-2:]
        if top2[1] - top2[0] > TOL * max(1.0, float(np.abs(lg).max())):
            assert int(np.argmax(lg)) == tok, i
            checked += 1
        x = o.run_position(o.embed(tok, len(prompt) + i), okv, list(range(len(okv))), pos=len(prompt) + i,
                           prefix=True)
    assert checked >= n_tok // 2


@pytest.mark.parametrize("stages,w,k", [(4, 8, 4), (8, 6, 3)])
def test_grouped_stage_forward_bitwise(stages, w, k):
    """tp_stages_forward (one grouped GEMM launch per layer slot over all
    same-device stages) == per-stage tp_stage_forward, bit for bit, every step;
    and the SpecPipe tokens equal the GPU greedy decode."""
    cfg, m, _ = tiny_model(layers=stages)
    prompt = [int(t) for t in np.random.default_rng(4).integers(0, cfg.vocab, 70)]
    n_tok = 20
    ref = tp.sequential_decode(m, prompt, n_tok + 3 * stages)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=5),
                              cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(ref))
    from paper_2504_04104_b200.pipeline import PipelineRunner

    rec = PipelineRunner(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=w, k=k), draft,
                         collect_trace=False, grouped=True)
    rec.children_log = []
    rec.prefill(prompt)
    while len(rec.emitted) < n_tok:
        rec.decode_step()
    assert rec.emitted == ref[: len(rec.emitted)]
    runs = {}
    for grouped in (True, False):
        r = PipelineRunner(m, tp.PipelineConfig(num_stages=stages), tp.BeamConfig(w=w, k=k), None,
                           collect_trace=False, grouped=grouped)
        r.prefill(prompt)
        outs = []
        for ch in rec.children_log:
            r.launch_compute()
            outs.append([None if s.out is None else s.out.cpu().clone() for s in r.stages])
            r.step(ch)
        runs[grouped] = (outs, list(r.emitted))
    assert runs[True][1] == runs[False][1] == rec.emitted
    for step, (a, b) in enumerate(zip(runs[True][0], runs[False][0])):
        for s, (x, y) in enumerate(zip(a, b)):
            assert (x is None) == (y is None), (step, s)
            if x is not None:
                assert torch.equal(x, y), (step, s)


def test_grouped_gemm_nine_stages_chunks():
    """More than 8 same-device stages: the group is split into launches of <= 8."""
    cfg, m, _ = tiny_model(layers=9)
    prompt = [int(t) for t in np.random.default_rng(8).integers(0, cfg.vocab, 20)]
    ref = tp.sequential_decode(m, prompt, 30)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.9, rank_decay=0.5, miss_prob=0.0, seed=2),
                              cfg.vocab)
    res = tp.run(m, tp.PipelineConfig(num_stages=9), tp.BeamConfig(w=3, k=3), draft, prompt, 20,
                 collect_trace=False)
    assert res.tokens == ref[:20]


def test_llama_long_context_invariance_and_oracle():
    """> 32 canonical chunks (2.2k-token prefix): siblings together == alone, a
    chain == sequential prefill (bitwise), and outputs within TOL of the oracle."""
    cfg, m, o = tiny_model()
    rng = np.random.default_rng(21)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, 2200)]
    base = KvCache(cfg.layers, cfg.hidden, capacity=2304)
    tp.model.prefill_rows(m, base, prompt)

    def fresh():
        c = KvCache(cfg.layers, cfg.hidden, capacity=2304)
        tp.model.prefill_rows(m, c, prompt)
        return c

    P = len(prompt)
    nodes = [(10 + i, int(rng.integers(cfg.vocab)), P, frozenset({10 + i})) for i in range(6)]
    together = forward_tree(m, fresh(), nodes).cpu()
    for i, nd in enumerate(nodes[:3]):
        alone = forward_tree(m, fresh(), [nd]).cpu()
        assert torch.equal(alone[0], together[i]), i
    okv = o.new_kv()
    x = None
    for pos, tok in enumerate(prompt + [nodes[0][1]]):
        x = o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
    got = together[0].numpy()
    assert float(np.abs(got - x).max()) <= TOL * max(1.0, float(np.abs(x).max()))


def test_attention_run_boundaries_ragged_prefixes():
    """Canonical runs of 8 chunks: nodes of ONE level with ragged verified
    prefixes (the shared kernel stops mid-run at floor(min P / 64); the tail
    continues that run and crosses further run boundaries with the prefix
    tails of the longer nodes), with scattered ancestor rows, are bit-identical
    to each node computed alone (its own c_shared, its own run split)."""
    cfg, m, _ = tiny_model()
    rng = np.random.default_rng(33)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, 1700)]
    cache = KvCache(cfg.layers, cfg.hidden, capacity=1792)
    tp.model.prefill_rows(m, cache, prompt)
    prefixes = [600, 1100, 1530, 513, 1024, 1650]
    rows, pos = [], []
    for P in prefixes:
        extra = sorted(rng.choice(np.arange(P + 1, 1700), size=5, replace=False).tolist())
        rows.append(np.concatenate([np.arange(P), np.asarray(extra)]).astype(np.int64))
        pos.append(P + len(extra))
    toks = [int(t) for t in rng.integers(0, cfg.vocab, len(prefixes))]
    uids = list(range(len(prefixes)))
    together = cache._forward(m, rows, None, toks, pos, None, False, uids, False).cpu()
    for i in range(len(prefixes)):
        alone = cache._forward(m, [rows[i]], None, [toks[i]], [pos[i]], None, False, [uids[i]], False).cpu()
        assert torch.equal(alone[0], together[i]), (i, prefixes[i])


def test_kv_capacity_growth_mid_decode_lossless():
    """Caches that start far too small grow by doubling (tp_stage_reserve:
    planes re-allocated and copied, attention scratch regrown) in the middle of
    a SpecPipe decode; the output stays identical to the greedy decode."""
    cfg, m, _ = tiny_model(layers=4)
    prompt = [int(t) for t in np.random.default_rng(12).integers(0, cfg.vocab, 40)]
    want = tp.sequential_decode(m, prompt, 24)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.05, seed=8),
                              cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(want))
    from paper_2504_04104_b200.pipeline import PipelineRunner

    r = PipelineRunner(m, tp.PipelineConfig(num_stages=4), tp.BeamConfig(w=12, k=4), draft, collect_trace=False,
                       kv_capacity=8)
    r.prefill(prompt)  # already grows 8 -> 64 rows
    caps0 = [s.kv._cap for s in r.stages]
    assert all(c >= len(prompt) for c in caps0)
    while len(r.emitted) < 24:
        r.decode_step()
    assert r.emitted[:24] == want
    assert any(s.kv._cap > c for s, c in zip(r.stages, caps0))  # and again while decoding


def test_gqa_attention_paths():
    """GQA (8 query heads over 2 KV heads): the group-staged shared-chunk and
    tail kernels keep batch invariance (siblings together == alone, bitwise),
    agree with the float32 oracle, and SpecPipe stays lossless."""
    shape = dict(vocab=512, hidden=256, layers=2, heads=8, kv_heads=2, ffn=512)
    cfg = LlamaConfig(**shape)
    m = LlamaModel(cfg, max_nodes=64)
    o = LlamaOracle(**shape)
    rng = np.random.default_rng(31)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, 150)]

    def fresh():
        c = KvCache(cfg.layers, cfg.hidden, capacity=256)
        tp.model.prefill_rows(m, c, prompt)
        return c

    P = len(prompt)
    nodes = [(10 + i, int(rng.integers(cfg.vocab)), P, frozenset({10 + i})) for i in range(9)]
    together = forward_tree(m, fresh(), nodes).cpu()
    for i, nd in enumerate(nodes[:4]):
        assert torch.equal(forward_tree(m, fresh(), [nd]).cpu()[0], together[i]), i
    okv = o.new_kv()
    x = None
    for pos, tok in enumerate(prompt + [nodes[0][1]]):
        x = o.run_position(o.embed(tok, pos), okv, list(range(len(okv))), pos=pos, prefix=True)
    assert float(np.abs(together[0].numpy() - x).max()) <= TOL * max(1.0, float(np.abs(x).max()))
    want = tp.sequential_decode(m, prompt[:30], 16)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.05, seed=3),
                              cfg.vocab)
    res = tp.run(m, tp.PipelineConfig(num_stages=2), tp.BeamConfig(w=8, k=4), draft, prompt[:30], 16,
                 collect_trace=False)
    assert res.tokens == want


@pytest.mark.gpu
def test_sharded_models_pipeline_lossless():
    """The `bench.py --gpus N` placement emulated on one GPU: per-stage shard model
    objects (layer ranges, embedding only on the first, head only on the last,
    LCG jump-ahead to their layers) driven as one pipeline, grouped per shard;
    tokens equal the single model's greedy decode and the staged oracle."""
    from paper_2504_04104_b200.pipeline import PipelineRunner, sequential_decode_staged, split_layers

    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=6, heads=2, kv_heads=1, ffn=512)
    full = tp.LlamaModel(cfg, max_nodes=64)
    stages = 6
    splits = split_layers(cfg.layers, stages)
    owner = [0, 0, 0, 1, 1, 1]  # two shards of three stages each
    shards = {}
    for o in sorted(set(owner)):
        mine = [splits[s] for s in range(stages) if owner[s] == o]
        lo, hi = mine[0][0], mine[-1][1]
        shards[o] = tp.LlamaModel(cfg, max_nodes=64, layer_range=(lo, hi), with_embed=lo == 0,
                                  with_head=hi == cfg.layers)
    per_stage = [shards[owner[s]] for s in range(stages)]
    prompt = [int(t) for t in np.random.default_rng(13).integers(0, cfg.vocab, 60)]
    ref = tp.sequential_decode(full, prompt, 30)
    assert sequential_decode_staged(per_stage, splits, prompt, 30) == ref
    for grouped in (True, False):
        draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.7, rank_decay=0.5, miss_prob=0.05, seed=4),
                                  cfg.vocab)
        draft.bind_reference(tuple(prompt) + tuple(ref))
        r = PipelineRunner(per_stage, tp.PipelineConfig(num_stages=stages, layer_splits=tuple(splits)),
                           tp.BeamConfig(w=8, k=4), draft, collect_trace=False, grouped=grouped)
        r.prefill(prompt)
        while len(r.emitted) < 20:
            r.decode_step()
        assert r.emitted[:20] == ref[:20], grouped
        r.close()


@pytest.mark.gpu
@pytest.mark.parametrize("threads,graphs", [(False, False), (True, False), (False, True)])
def test_cross_shard_protocol_on_one_gpu(threads, graphs, monkeypatch):
    """The stage-per-GPU step protocol (send-before-verify hand-offs by
    tp_peer_copy, K4's result mirrored to every shard by tp_result_mirror,
    per-shard tp_prune_device with receiver-side compaction of the hand-offs)
    exercised on one GPU with one stream per shard: tokens equal the greedy
    decode, and every step's device keep lists equal the single-shard run's."""
    import paper_2504_04104_b200.pipeline as PL
    from paper_2504_04104_b200.pipeline import PipelineRunner, split_layers

    # threads: each shard's launches and K3 issued from its own host thread (the
    # multi-device mode), forced on one device
    monkeypatch.setattr(PL, "_SHARD_THREADS_FORCE", threads)
    # graphs: each shard's lone forward captured and replayed as a CUDA graph (TP_GRAPH)
    from paper_2504_04104_b200 import _lib

    _lib.check(_lib.lib().tp_debug_attn_knob(5, int(graphs)))
    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=6, heads=2, kv_heads=1, ffn=512)
    full = tp.LlamaModel(cfg, max_nodes=64)
    stages = 6
    splits = split_layers(cfg.layers, stages)
    owner = [0, 0, 1, 1, 2, 2]  # three shards of two stages each
    shards = {}
    for o in sorted(set(owner)):
        mine = [splits[s] for s in range(stages) if owner[s] == o]
        lo, hi = mine[0][0], mine[-1][1]
        shards[o] = tp.LlamaModel(cfg, max_nodes=64, layer_range=(lo, hi), with_embed=lo == 0,
                                  with_head=hi == cfg.layers)
    per_stage = [shards[owner[s]] for s in range(stages)]
    prompt = [int(t) for t in np.random.default_rng(21).integers(0, cfg.vocab, 60)]
    ref = tp.sequential_decode(full, prompt, 40)

    def run(models, shard_streams):
        draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=5),
                                  cfg.vocab)
        draft.bind_reference(tuple(prompt) + tuple(ref))
        r = PipelineRunner(models, tp.PipelineConfig(num_stages=stages, layer_splits=tuple(splits)),
                           tp.BeamConfig(w=8, k=4), draft, collect_trace=False, shard_streams=shard_streams)
        r.capture_device_keeps = []
        r.prefill(prompt)
        keeps = []
        while len(r.emitted) < 28:
            r.decode_step()
            keeps.append([list(x) for x in r.last_keeps] if r.last_keeps else None)
        import torch

        torch.cuda.synchronize()
        return r, keeps

    r1, k1 = run(full, False)
    r2, k2 = run(per_stage, True)
    assert r2.cross and not r1.cross
    assert r2.emitted[:28] == ref[:28] == r1.emitted[:28]
    assert k1 == k2
    dev1 = [[int(b[0])] + b[2:2 + int(b[0])].tolist() for b in (x.cpu() for x in r1.capture_device_keeps[-1])]
    dev2 = [[int(b[0])] + b[2:2 + int(b[0])].tolist() for b in (x.cpu() for x in r2.capture_device_keeps[-1])]
    assert dev1 == dev2
    r1.close()
    r2.close()
    _lib.check(_lib.lib().tp_debug_attn_knob(5, 0))


@pytest.mark.gpu
@pytest.mark.parametrize("cross", [False, True])
def test_draft_model_stage(cross):
    """The draft-model forward (BASELINE configs 2/4) inside the step: the draft's
    cache mirrors stage 1's rows through every prune, tokens stay lossless, and
    the draft's logits for a tree node equal a causal forward of the draft over
    that node's path (prompt + ancestors + node), i.e. the tree masking holds."""
    from paper_2504_04104_b200.pipeline import PipelineRunner, split_layers

    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
    dcfg = tp.LlamaConfig(vocab=512, hidden=256, layers=1, heads=2, kv_heads=2, ffn=512, seed=9)
    full = tp.LlamaModel(cfg, max_nodes=64)
    dm = tp.LlamaModel(dcfg, max_nodes=64)
    stages = 4
    splits = split_layers(cfg.layers, stages)
    models = full
    if cross:
        models = [tp.LlamaModel(cfg, max_nodes=64, layer_range=sp, with_embed=sp[0] == 0,
                                with_head=sp[1] == cfg.layers) for sp in splits]
    prompt = [int(t) for t in np.random.default_rng(33).integers(0, cfg.vocab, 40)]
    ref = tp.sequential_decode(full, prompt, 30)
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=2), cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(ref))
    r = PipelineRunner(models, tp.PipelineConfig(num_stages=stages, layer_splits=tuple(splits)),
                       tp.BeamConfig(w=6, k=3), draft, collect_trace=False, shard_streams=cross, draft_model=dm)
    r.capture_draft = []
    r.prefill(prompt)
    checked = 0
    while len(r.emitted) < 20:
        r.decode_step()
        s1, dk = r.stages[0].kv, r.draft_stage.kv
        assert len(s1) == len(dk) and np.array_equal(s1._uid, dk._uid) and np.array_equal(s1._pref, dk._pref)
        if r.capture_draft and checked < 6 and r.tree is not None:
            uids, pos, logits = r.capture_draft[-1]
            node = len(uids) - 1  # the level's last node: its path from the tree
            path = []
            u = uids[node]
            if u in r.tree._uid_index:
                i = r.tree._uid_index[u]
                anc = np.flatnonzero(tp.tree.mask_row(r.tree, i).bits)
                path = [int(r.tree.tokens[j]) for j in anc]  # root .. node (root = last verified token)
                seq = r.verified[: pos[node] - len(path) + 1] + path
                assert len(seq) == pos[node] + 1
                cache = tp.KvCache(dcfg.layers, dcfg.hidden)
                rows = tp.model.prefill_rows(dm, cache, seq)
                want = dm.logits_many(rows[-1:])[0].float().cpu()
                got = logits[node]
                assert float((got - want).abs().max()) <= 1e-4 * max(1.0, float(want.abs().max()))
                checked += 1
    import torch

    torch.cuda.synchronize()
    assert r.emitted[:20] == ref[:20]
    assert checked >= 2
    r.release()


@pytest.mark.gpu
def test_cross_shard_graphs_lossless():
    """One shard per stage (the --gpus 8 placement) on shard streams with the
    CUDA-graph mode on: every lone stage forward is a graph replay, and tokens and
    device keep lists equal the same run without graphs."""
    import ctypes as C

    from paper_2504_04104_b200 import _lib
    from paper_2504_04104_b200.pipeline import PipelineRunner, split_layers

    cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=6, heads=2, kv_heads=1, ffn=512)
    full = tp.LlamaModel(cfg, max_nodes=64)
    stages = 6
    splits = split_layers(cfg.layers, stages)
    shards = [tp.LlamaModel(cfg, max_nodes=64, layer_range=sp, with_embed=sp[0] == 0, with_head=sp[1] == cfg.layers)
              for sp in splits]
    prompt = [int(t) for t in np.random.default_rng(22).integers(0, cfg.vocab, 60)]
    ref = tp.sequential_decode(full, prompt, 34)

    def run(graphs):
        _lib.check(_lib.lib().tp_debug_attn_knob(5, int(graphs)))
        draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=0.6, rank_decay=0.5, miss_prob=0.1, seed=7),
                                  cfg.vocab)
        draft.bind_reference(tuple(prompt) + tuple(ref))
        r = PipelineRunner(shards, tp.PipelineConfig(num_stages=stages, layer_splits=tuple(splits)),
                           tp.BeamConfig(w=8, k=4), draft, collect_trace=False, shard_streams=True)
        r.prefill(prompt)
        keeps = []
        while len(r.emitted) < 24:
            r.decode_step()
            keeps.append([list(x) for x in r.last_keeps] if r.last_keeps else None)
        torch.cuda.synchronize()
        r.release()
        _lib.check(_lib.lib().tp_debug_attn_knob(5, 0))
        return r.emitted[:24], keeps

    n0 = C.c_int64()
    _lib.check(_lib.lib().tp_graph_launches(C.byref(n0)))
    e_graph, k_graph = run(True)
    n1 = C.c_int64()
    _lib.check(_lib.lib().tp_graph_launches(C.byref(n1)))
    e_plain, k_plain = run(False)
    assert e_graph == e_plain == ref[:24]
    assert k_graph == k_plain
    assert n1.value - n0.value > 24  # lone stage forwards actually ran as graphs


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_pipeline_lossless_randomized(seed):
    """Losslessness (acceptance 1) over randomized configurations: stage count,
    beam width / branching, MHA / GQA, a fused draft model, one shard per stage on
    shard streams (the stage-per-GPU protocol) or one model object — the pipeline's
    tokens always equal the GPU greedy decode."""
    from paper_2504_04104_b200.pipeline import PipelineRunner, split_layers

    rng = np.random.default_rng(100 + seed)
    heads, kv = [(2, 1), (2, 2), (4, 1)][seed % 3]
    layers = int(rng.integers(4, 9))
    stages = int(rng.integers(2, min(6, layers) + 1))
    cfg = tp.LlamaConfig(vocab=512, hidden=128 * heads, layers=layers, heads=heads, kv_heads=kv, ffn=512,
                         seed=seed)
    full = tp.LlamaModel(cfg, max_nodes=64)
    splits = split_layers(layers, stages)
    sharded = bool(seed % 2)
    models = ([tp.LlamaModel(cfg, max_nodes=64, layer_range=sp, with_embed=sp[0] == 0, with_head=sp[1] == layers)
               for sp in splits] if sharded else full)
    dm = (tp.LlamaModel(tp.LlamaConfig(vocab=512, hidden=256, layers=1, heads=2, kv_heads=2, ffn=256, seed=50 + seed),
                        max_nodes=64) if seed % 3 != 1 else None)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, int(rng.integers(20, 90)))]
    ref = tp.sequential_decode(full, prompt, 30)
    w, k = int(rng.integers(2, 17)), int(rng.integers(2, 7))
    draft = tp.SyntheticDraft(tp.SyntheticDraftConfig(top1_hit=float(rng.uniform(0.3, 0.8)), rank_decay=0.5,
                                                      miss_prob=float(rng.uniform(0.0, 0.2)), seed=seed), cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(ref))
    r = PipelineRunner(models, tp.PipelineConfig(num_stages=stages, layer_splits=tuple(splits)), tp.BeamConfig(w=w, k=k),
                       draft, collect_trace=False, shard_streams=sharded, draft_model=dm)
    r.prefill(prompt)
    while len(r.emitted) < 20:
        r.decode_step()
    torch.cuda.synchronize()
    assert r.emitted[:20] == ref[:20], (seed, stages, w, k, heads, kv, sharded, dm is not None)
    r.release()


@pytest.mark.gpu
def test_llama_max_nodes_limit():
    """A Llama forward is one K2 GEMM over a member's rows (<= 256): larger
    max_nodes is refused when the model is created, not at the first forward."""
    from paper_2504_04104_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        LlamaModel(LlamaConfig(**TINY), max_nodes=257)
    LlamaModel(LlamaConfig(**TINY), max_nodes=256)
