"""Llama-arch oracle: numpy float32 restatement of the B200 Llama step (TEST ONLY).

PARITY UNPINNED for the arithmetic: the reference has no Llama model (its
only decoder is the float64 ToyModel).  What *is* pinned is shared with the
toy oracle: the weight stream (oracle/lcg.py), the tree / KV semantics
(`model.py:157-163,312-349` — prefix rows, ancestors, self last, recompute
mode), verification and pruning (oracle/pipeline.py).

Numerics mirrored from csrc/llama.cu and csrc/attn.cu:
  weights      f64 LCG sample * sqrt(3/fan_in)/0.1 -> f32 -> bf16 (RNE)
  rmsnorm      r = 1/sqrt(mean(x^2) + eps) (f32); h = bf16(x*r)
  projections  bf16 inputs, f32 accumulation; residual stream f32
  rope         HF rotate-half, angle = pos * theta^(-2i/128) in f64
  attention    bf16 q/k/v, f32 softmax, P rounded to bf16 before P.V
  swiglu       bf16(g / (1 + exp(-g)) * u)
The GPU accumulates in different orders (tensor-core tiles, online softmax
over 64-slot chunks), so comparisons use a stated tolerance.
"""

from __future__ import annotations

import numpy as np

from .lcg import uniform_stream
from .toy import OracleKv

F32 = np.float32


def bf16(x) -> np.ndarray:
    """Round float32 values to bfloat16 precision (round-to-nearest-even), kept as float32."""
    a = np.ascontiguousarray(x, dtype=F32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(F32).reshape(a.shape)


class LlamaOracle:
    def __init__(self, vocab, hidden, layers, heads, kv_heads, ffn, seed=0, rope_theta=10000.0, norm_eps=1e-5,
                 weight_scale=True, layer_range=None, with_head=True):
        self.vocab, self.hidden, self.layers = vocab, hidden, layers
        self.heads, self.kv_heads, self.ffn = heads, kv_heads, ffn
        self.theta, self.eps = rope_theta, norm_eps
        d, q, kv, f = hidden, heads * 128, kv_heads * 128, ffn
        per_layer = d * q + 2 * d * kv + q * d + 3 * d * f
        lo, hi = layer_range if layer_range is not None else (0, layers)
        self.layer_range = (lo, hi)

        def mat(start, rows, cols, fan_in):
            u = uniform_stream(seed, rows * cols, start).reshape(rows, cols)
            scale = np.sqrt(3.0 / fan_in) / 0.1 if weight_scale else 1.0
            return bf16((u * scale).astype(F32))

        self.embedding = bf16(uniform_stream(seed, vocab * d, 0).astype(F32)).reshape(vocab, d)
        self.blocks = {}
        for layer in range(lo, hi):
            off = vocab * d + layer * per_layer
            b = {}
            for name, rows, cols, fan in (("wq", d, q, d), ("wk", d, kv, d), ("wv", d, kv, d), ("wo", q, d, q),
                                          ("wg", d, f, d), ("wu", d, f, d), ("wd", f, d, f)):
                b[name] = mat(off, rows, cols, fan)
                off += rows * cols
            self.blocks[layer] = b
        self.lm_head = mat(vocab * d + layers * per_layer, d, vocab, d) if with_head else None
        i = np.arange(64, dtype=np.float64)
        self._inv = self.theta ** (-2.0 * i / 128.0)

    # -- pieces ---------------------------------------------------------------
    def norm(self, x):
        x = x.astype(F32)
        r = F32(1.0) / np.sqrt(np.mean(x * x, dtype=F32) + F32(self.eps), dtype=F32)
        return bf16(x * r)

    def rope(self, y, pos):
        ang = pos * self._inv
        c, s = np.cos(ang).astype(F32), np.sin(ang).astype(F32)
        y = y.reshape(-1, 128)
        y1, y2 = y[:, :64], y[:, 64:]
        return np.concatenate([y1 * c - y2 * s, y2 * c + y1 * s], axis=1).reshape(-1)

    def embed(self, token, pos):
        return self.embedding[token].astype(F32).copy()

    def logits(self, x):
        return self.norm(x) @ self.lm_head

    def greedy(self, x):
        return int(np.argmax(self.logits(x)))

    def block(self, layer, x, kv: OracleKv, rows, append, pos):
        w = self.blocks[layer]
        h = self.norm(x)
        q = self.rope(h @ w["wq"], pos)
        k = self.rope(h @ w["wk"], pos)
        v = h @ w["wv"]
        qb, kb, vb = bf16(q), bf16(k), bf16(v)
        if append:
            kv.put(layer, kb, vb)
        ks = np.concatenate([kv.k_rows(layer, rows).reshape(-1, kb.size), kb[None, :]])
        vs = np.concatenate([kv.v_rows(layer, rows).reshape(-1, vb.size), vb[None, :]])
        group = self.heads // self.kv_heads
        out = np.empty(self.heads * 128, dtype=F32)
        scale = F32(1.0 / np.sqrt(128.0))
        for hh in range(self.heads):
            kh = hh // group
            kmat = ks[:, kh * 128:(kh + 1) * 128]
            vmat = vs[:, kh * 128:(kh + 1) * 128]
            s = (kmat @ qb[hh * 128:(hh + 1) * 128]) * scale
            p = np.exp(s - s.max()).astype(F32)
            out[hh * 128:(hh + 1) * 128] = (bf16(p) @ vmat) / p.sum(dtype=F32)
        x = x + bf16(out) @ w["wo"]
        h2 = self.norm(x)
        g = h2 @ w["wg"]
        u = h2 @ w["wu"]
        a = bf16((g / (F32(1.0) + np.exp(-g))) * u)
        return (x + a @ w["wd"]).astype(F32)

    def run_position(self, x, kv, rows, layer_range=None, append=True, uid=-1, pos=0, prefix=False):
        lo, hi = layer_range if layer_range is not None else self.layer_range
        if append:
            kv.open_row(uid, pos, prefix)
        x = np.asarray(x, dtype=F32)
        for layer in range(lo, hi):
            x = self.block(layer, x, kv, rows, append, pos)
        return x

    def new_kv(self) -> OracleKv:
        return OracleKv(self.layers, self.kv_heads * 128)
