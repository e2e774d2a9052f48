"""Llama parity at the BENCHMARKED shapes (BASELINE.json configs 2-4).

A real stage step is pushed through a 1-2 layer slice of the 7B (32x128 MHA),
13B (40 heads) and 70B (64/8 GQA, d=8192, f=28672) shapes:

  prompt prefill (512 / 512 / 4096 tokens)  ->  a w=16 first tree level  ->
  a w=64 second level (4 children per node)  ->  verification hit on one
  level-1 child: promote + prune (row-or-column keep rule, pipeline.py:341-353)
  ->  a w=64 third level over the pruned cache  ->  LM-head logits.

Three kinds of evidence, each with its own stated bound:

1. **Per kernel, tight** (the level-2 forward, captured with tp_debug_dump):
   every kernel's output against a float64 recomputation from that kernel's
   own GPU inputs — the bf16 operand of the folded input RMSNorm, QKV+RMSNorm
   scale+RoPE (queries and the K/V rows written
   to the cache), tree attention with the ancestor mask (prefix ∪ ancestors,
   self last), o-projection + residual, RMSNorm, gate/up + SwiGLU, down +
   residual.  bf16 outputs: >= 99.9 % of elements within one bf16 ulp of the
   float64 value; attention (P is rounded to bf16 before P·V, the output to
   bf16): rms error <= ATT_TOL of the exact softmax; float32 outputs: max
   error <= 5e-5 of the row scale.  Controls at the same level: the attention
   reference with one ancestor row swapped must be >= 4x ATT_TOL away, the
   query RoPE'd at position+1 >= 5 % rms away.
2. **End to end vs the float32 oracle** (oracle/llama.py, itself validated with
   the reference's acceptance-2/3 logic in test_oracle_llama.py): keep lists
   bit-exact, the K/V rows surviving compaction bit-identical to the same rows
   before it, hidden states / K rows / logits within TOL_MAX (max) and TOL_RMS
   (rms) of the oracle's scale, greedy tokens equal where the oracle's top-1
   margin exceeds the bound.  The bound is measured, not guessed: tensor-core
   fp32 accumulation differs from numpy's by ~1e-6..1e-5 relative, which flips
   ~0.1 % of each bf16 re-rounding (v, h, the SwiGLU product) by one ulp, and
   every flip in a normalised row feeds all outputs of the next GEMM — the
   chain reaches ~1e-3 rms per layer (profiles/r02_llama_shape_parity.txt).
3. **End-to-end controls**: the GPU's level-3 output is compared with the
   oracle run under a wrong RoPE position and under a wrong ancestor row; both
   must be at least 2x farther than the correct oracle (at a 4k prefix one
   ancestor row is 1/4097 of the attention mass, so the kernel-level control
   above is the sharp one there).
"""

import copy
import json
import os

import numpy as np
import pytest
import torch

from oracle.llama import LlamaOracle

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2504_04104_b200")
from paper_2504_04104_b200 import _lib  # noqa: E402
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, forward_tree, prefill_rows  # noqa: E402

TOL_MAX = 2e-2   # end to end vs the oracle (measured <= 7.4e-3 at 7B / 13B)
TOL_RMS = 1e-2   # (measured <= 6.7e-3)
ATT_TOL = 3.5e-3  # tree attention vs exact softmax from the kernel's own Q/K/V (measured 2.1e-3:
                 # the bf16 output rounding alone is ~1.6e-3 rms)

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


def within_ulps(got, ref, k):
    """Fraction of bf16 values within k bf16 ulps (at the float64 value's binade) of ref."""
    ref = ref.double()
    e = torch.floor(torch.log2(ref.abs().clamp_min(1e-30)))
    ulp = torch.pow(2.0, e - 7)
    return float(((got.double() - ref).abs() <= k * ulp * 1.0001).double().mean())


def bfr(t):
    return t.float().to(torch.bfloat16).double()


class Weights:
    """Layer-`lo` weights read back from the device model, as float64 on the GPU."""

    def __init__(self, model, cfg, layer):
        d, q, kv, f = cfg.hidden, cfg.heads * 128, cfg.kv_heads * 128, cfg.ffn

        def W(which, shape, lyr=layer):
            u = model.read_tensor(which, lyr).view(np.uint16)
            return torch.from_numpy(as_f32(u).reshape(shape)).cuda().double()

        qkv = W(1, (q + 2 * kv, d))
        self.wq, self.wk, self.wv = qkv[:q], qkv[q:q + kv], qkv[q + kv:]
        self.wo = W(4, (d, q))
        gu = W(5, (2 * f // 128, 2, 64, d))
        self.wg, self.wu = gu[:, 0].reshape(f, d), gu[:, 1].reshape(f, d)
        self.wd = W(7, (d, f))
        self.emb = W(0, (cfg.vocab, d), 0)
        self.eps = cfg.norm_eps
        self.theta = cfg.rope_theta

    def norm(self, x):
        return x * torch.rsqrt((x * x).mean(dim=1, keepdim=True) + self.eps)

    def rscale(self, x):
        """The folded RMSNorm's per-row scale r (the GEMMs consume bf16(x), then scale by r)."""
        return torch.rsqrt((x * x).mean(dim=1, keepdim=True) + self.eps)

    def rope(self, y, pos):
        i = torch.arange(64, dtype=torch.float64, device=y.device)
        ang = torch.as_tensor(pos, dtype=torch.float64, device=y.device)[:, None] * self.theta ** (-2.0 * i / 128.0)
        c, s = torch.cos(ang).float().double()[:, None, :], torch.sin(ang).float().double()[:, None, :]
        y = y.reshape(y.shape[0], -1, 128)
        y1, y2 = y[..., :64], y[..., 64:]
        return torch.cat([y1 * c - y2 * s, y2 * c + y1 * s], dim=2).reshape(y.shape[0], -1)


def kernel_checks(cfg, W, dump, n, x_in, pos, rows, wrong_rows, kc, vc, self_rows):
    """Per-kernel float64 parity of one captured forward (see module doc, item 1)."""
    d, q, kv, f = cfg.hidden, cfg.heads * 128, cfg.kv_heads * 128, cfg.ffn
    o = 0

    def take(nbytes, dt, shape):
        nonlocal o
        t = dump[o:o + nbytes].view(dt).reshape(shape)
        o += nbytes
        return t.float().double() if dt == torch.bfloat16 else t.double()

    Xd = take(n * d * 2, torch.bfloat16, (n, d))
    Xq = take(n * q * 2, torch.bfloat16, (n, q))
    Xo = take(n * q * 2, torch.bfloat16, (n, q))
    xo = take(n * d * 4, torch.float32, (n, d))
    Xd2 = take(n * d * 2, torch.bfloat16, (n, d))
    Xf = take(n * f * 2, torch.bfloat16, (n, f))
    xd = take(n * d * 4, torch.float32, (n, d))
    res = {}
    # RMSNorm is folded into the GEMMs: the operand is bf16(x), the projection is scaled by r
    r_in = W.rscale(x_in)
    res["norm_operand_in"] = within_ulps(Xd, x_in, 0.5)  # bf16(x): round to nearest
    res["q_rope"] = within_ulps(Xq, W.rope((Xd @ W.wq.t()) * r_in, pos), 1)
    res["k_rope"] = within_ulps(kc[self_rows], W.rope((Xd @ W.wk.t()) * r_in, pos), 1)
    res["v"] = within_ulps(vc[self_rows], (Xd @ W.wv.t()) * r_in, 1)
    g = cfg.heads // cfg.kv_heads
    att = torch.empty((n, q), dtype=torch.float64, device="cuda")
    att_b = torch.empty_like(att)
    for i in range(n):
        r = torch.as_tensor(list(rows[i]) + [self_rows[i]], device="cuda")
        K = kc[r].reshape(-1, cfg.kv_heads, 128)
        V = vc[r].reshape(-1, cfg.kv_heads, 128)
        Q = Xq[i].reshape(cfg.kv_heads, g, 128)
        s = torch.einsum("kgd,rkd->kgr", Q, K) / np.sqrt(128.0)
        p = torch.softmax(s, dim=2)
        att[i] = torch.einsum("kgr,rkd->kgd", p, V).reshape(-1)
        pb = bfr(torch.exp(s - s.amax(dim=2, keepdim=True)))  # P rounded to bf16 before P.V, as the kernel
        att_b[i] = (torch.einsum("kgr,rkd->kgd", pb, V) / torch.exp(s - s.amax(dim=2, keepdim=True)).float()
                    .double().sum(dim=2, keepdim=True)).reshape(-1)
    res["attention_rel_rms"] = rel_err(Xo.cpu(), att.cpu())[1]
    res["attention_within_2ulp_of_bf16P"] = within_ulps(Xo, att_b, 2)  # informational
    res["o_proj_resid"] = rel_err(xo.cpu(), (x_in + Xo @ W.wo.t()).cpu())[0]
    r_o = W.rscale(xo)
    res["norm_operand_post"] = within_ulps(Xd2, xo, 0.5)
    gg, uu = (Xd2 @ W.wg.t()) * r_o, (Xd2 @ W.wu.t()) * r_o
    res["swiglu"] = within_ulps(Xf, gg / (1 + torch.exp(-gg)) * uu, 1)
    res["down_resid"] = rel_err(xd.cpu(), (xo + Xf @ W.wd.t()).cpu())[0]
    # controls at kernel level: the same references under a wrong ancestor row / RoPE position
    wrong = torch.empty_like(att)
    for i in range(n):
        r = torch.as_tensor(list(wrong_rows[i]) + [self_rows[i]], device="cuda")
        K = kc[r].reshape(-1, cfg.kv_heads, 128)
        V = vc[r].reshape(-1, cfg.kv_heads, 128)
        s = torch.einsum("kgd,rkd->kgr", Xq[i].reshape(cfg.kv_heads, g, 128), K) / np.sqrt(128.0)
        wrong[i] = torch.einsum("kgr,rkd->kgd", torch.softmax(s, dim=2), V).reshape(-1)
    res["control_attention_wrong_row_rel_rms"] = rel_err(Xo.cpu(), wrong.cpu())[1]
    res["control_q_rope_pos+1_rel_rms"] = rel_err(Xq.cpu(), W.rope((Xd @ W.wq.t()) * r_in,
                                                                  [p + 1 for p in pos]).cpu())[1]
    for k, v in res.items():
        if k in ("o_proj_resid", "down_resid"):
            assert v <= 5e-5, (k, v)
        elif k == "attention_rel_rms":
            assert v <= ATT_TOL, (k, v)
        elif k == "control_attention_wrong_row_rel_rms":
            assert v >= 4 * ATT_TOL, (k, v)
        elif k == "control_q_rope_pos+1_rel_rms":
            assert v >= 0.05, (k, v)  # vs <= 1 ulp (~2e-3) at the right position
        elif k != "attention_within_2ulp_of_bf16P":
            assert v >= 0.999, (k, v)
    return res


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
    g1 = forward_tree(model, cache, w1, layer_range=(lo, hi))
    check("level1", g1, orc.forward_level(okv, w1))

    # level 2 with every first-layer intermediate captured for the per-kernel checks
    d, q, f = cfg.hidden, cfg.heads * 128, cfg.ffn
    dump = torch.zeros(64 * (d * 2 + q * 2 * 2 + d * 4 + d * 2 + f * 2 + d * 4), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().tp_debug_dump(dump.data_ptr()))
    g2 = forward_tree(model, cache, w2, layer_range=(lo, hi))
    torch.cuda.synchronize()
    check("level2", g2, orc.forward_level(okv, w2))
    W = Weights(model, cfg, lo)
    kc = torch.from_numpy(as_f32(cache.keys[lo])).cuda().double()
    vc = torch.from_numpy(as_f32(cache.values[lo])).cuda().double()
    x_in = W.emb[torch.as_tensor([nd[1] for nd in w2], device="cuda")]
    rows = [list(range(P)) + [P + j // 4] for j in range(64)]
    wrong_rows = [list(range(P)) + [P + (j // 4 + 1) % 16] for j in range(64)]
    kern = kernel_checks(cfg, W, dump, 64, x_in, [P + 1] * 64, rows, wrong_rows, kc, vc,
                         [P + 16 + j for j in range(64)])

    k_before = cache.keys[lo]
    check("k_rows", as_f32(k_before[P:]), okv.keys(lo)[P:])

    # verification hit on level-1 child 5: promote the chain, prune to row-or-column
    child = 1000 + 5
    keep = {child} | {2000 + j for j in range(64) if j // 4 == 5}
    cache.promote({child})
    cache.prune(keep)
    okv.promote({child})
    okeep = okv.keep_rows(keep)
    okv.restrict(okeep)
    assert cache.last_keep == okeep
    assert cache.uids == okv.uids and cache.positions == okv.positions
    assert np.array_equal(cache.keys[lo], k_before[okeep])  # compaction moves rows bit for bit

    # level 3 over the pruned cache: 64 grandchildren of the 4 surviving level-2 nodes
    surv = [2000 + j for j in range(64) if j // 4 == 5]
    w3 = [(3000 + j, int(rng.integers(cfg.vocab)), P + 2, frozenset({surv[j % 4], 3000 + j})) for j in range(64)]
    g3 = forward_tree(model, cache, w3, layer_range=(lo, hi))
    okv_pre = copy.deepcopy(okv)
    o3 = orc.forward_level(okv, w3)
    check("level3_after_prune", g3, o3)

    # sensitivity controls: wrong RoPE position / wrong ancestor row are far outside the bound
    g3n = g3.detach().float().cpu().numpy()
    bad_pos = [(u, t, p + 1, a) for u, t, p, a in w3]
    bad_anc = [(3000 + j, w3[j][1], P + 2, frozenset({surv[(j + 1) % 4], 3000 + j})) for j in range(64)]
    control = {}
    for tag, lvl in (("rope_pos+1", bad_pos), ("wrong_ancestor", bad_anc)):
        control[tag] = rel_err(g3n, orc.forward_level(copy.deepcopy(okv_pre), lvl))
        # the GPU sits far closer to the right semantics than to the wrong one
        assert control[tag][1] >= 2 * errs["level3_after_prune"][1], (tag, control[tag])

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
        fh.write(json.dumps({"shape": name, "layers": [lo, hi], "prompt": P, "e2e_errors_max_rms": errs,
                             "per_kernel": kern, "controls_max_rms": control, "argmax_checked": agreed}) + "\n")
    print(name, json.dumps({"e2e": errs, "kernels": kern, "controls": control}))
