"""Llama-arch oracle: numpy float32 restatement of the B200 Llama step (TEST ONLY).

PARITY UNPINNED for the arithmetic: the reference has no Llama model (its
only decoder is the float64 ToyModel).  What *is* pinned is shared with the
toy oracle: the weight stream (oracle/lcg.py), the tree / KV semantics
(`model.py:157-163,312-349` — prefix rows, ancestors, self last, recompute
mode), verification and pruning (oracle/pipeline.py).

Numerics mirrored from csrc/llama.cu and csrc/attn.cu:
  weights      f64 LCG sample * sqrt(3/fan_in)/0.1 -> f32 -> bf16 (RNE)
  rmsnorm      r = 1/sqrt(mean(x^2) + eps) (f32), folded into the GEMMs as the GPU does:
               projections of the normed rows = (bf16(x) . W) * r; the LM head's
               input keeps h = bf16(x*r)
  projections  bf16 inputs, f32 accumulation; residual stream f32
  rope         HF rotate-half, angle = pos * theta^(-2i/128) in f64
  attention    bf16 q/k/v, f32 softmax, P rounded to bf16 before P.V
  swiglu       bf16(g / (1 + exp(-g)) * u)  (the GPU: ex2.approx / rcp.approx, a few ulp before the bf16 rounding)
The GPU accumulates in different orders (tensor-core tiles, online softmax
over 64-slot chunks), so comparisons use a stated tolerance.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .lcg import uniform_stream
from .toy import OracleKv

F32 = np.float32


class DenseKv(OracleKv):
    """``OracleKv`` semantics (reference KvCache, `model.py:105-204`) with the
    per-layer K/V rows held in growable dense arrays, so the batched oracle
    forwards below can gather thousands of rows per node cheaply."""

    def __init__(self, layers: int, width: int, capacity: int = 256):
        super().__init__(layers, width)
        self.k = [np.zeros((capacity, width), F32) for _ in range(layers)]
        self.v = [np.zeros((capacity, width), F32) for _ in range(layers)]
        self.filled = [0] * layers

    def _grow(self, layer, rows):
        cap = self.k[layer].shape[0]
        if rows <= cap:
            return
        while cap < rows:
            cap *= 2
        for store in (self.k, self.v):
            new = np.zeros((cap, self.hidden), F32)
            new[: self.filled[layer]] = store[layer][: self.filled[layer]]
            store[layer] = new

    def put_many(self, layer, k, v):
        n0 = self.filled[layer]
        self._grow(layer, n0 + len(k))
        self.k[layer][n0 : n0 + len(k)] = k
        self.v[layer][n0 : n0 + len(v)] = v
        self.filled[layer] = n0 + len(k)

    def put(self, layer, k, v):
        self.put_many(layer, k[None, :], v[None, :])

    def _rows(self, store, rows):  # store is a dense array here
        return store[np.asarray(rows, dtype=np.int64)] if len(rows) else np.empty((0, self.hidden), F32)

    def k_rows(self, layer, rows):
        return self._rows(self.k[layer], rows)

    def v_rows(self, layer, rows):
        return self._rows(self.v[layer], rows)

    def keys(self, layer):
        return self.k[layer][: self.filled[layer]]

    def values(self, layer):
        return self.v[layer][: self.filled[layer]]

    def allowed(self, ancestors):
        anc = np.fromiter((int(a) for a in ancestors), dtype=np.int64)
        u = np.asarray(self.uids, dtype=np.int64)
        return np.flatnonzero(np.asarray(self.prefix, dtype=bool) | np.isin(u, anc)).tolist()

    def restrict(self, keep):
        keep = np.asarray(keep, dtype=np.int64)
        for layer in range(len(self.k)):
            if self.filled[layer]:
                self.k[layer][: keep.size] = self.k[layer][keep]
                self.v[layer][: keep.size] = self.v[layer][keep]
                self.filled[layer] = keep.size
        self.uids = [self.uids[i] for i in keep]
        self.positions = [self.positions[i] for i in keep]
        self.prefix = [self.prefix[i] for i in keep]


def _butterfly32(v: np.ndarray) -> np.ndarray:
    """A warp's xor-butterfly sum over the last axis (32 lanes), float32 adds in the
    GPU's order (every lane ends with the same value)."""
    v = v.astype(F32)
    lanes = np.arange(32)
    for o in (16, 8, 4, 2, 1):
        v = (v + v[..., lanes ^ o]).astype(F32)
    return v[..., 0]


def rms_scale_gpu_order(x: np.ndarray, eps: float) -> np.ndarray:
    """r = 1/sqrt(mean(x^2) + eps) per row, with the GPU's summation order
    (csrc/gemm_tc.h tile_sumsq and gemm_tc.cu norm_scale_from_partials): per
    128-column tile, lane l takes columns 4l..4l+3 as x0*x0 then three fused
    multiply-adds, a 32-lane butterfly gives the tile's partial; lane l then sums
    partials l, l+32, ... in order and a second butterfly gives the total."""
    x = np.atleast_2d(np.asarray(x, dtype=F32))
    n, d = x.shape
    q = x.reshape(n, d // 128, 32, 4).astype(np.float64)
    s = (q[..., 0] * q[..., 0]).astype(F32)
    for j in (1, 2, 3):  # fma: exact product + sum in float64, one rounding to float32
        s = (q[..., j] * q[..., j] + s.astype(np.float64)).astype(F32)
    part = _butterfly32(s)  # [n, tiles]
    tiles = part.shape[1]
    lanes = np.zeros((n, 32), dtype=F32)
    for i in range(tiles):
        lanes[:, i % 32] = (lanes[:, i % 32] + part[:, i]).astype(F32)
    ss = _butterfly32(lanes)
    return (F32(1.0) / np.sqrt((ss / F32(d)).astype(F32) + F32(eps), dtype=F32)).astype(F32)


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

        def mat(start, rows, cols, fan_in, scaled=True):
            # chunked over host threads (numpy ufuncs release the GIL); every
            # chunk is the exact stream slice [start+off, start+off+len)
            scale = np.sqrt(3.0 / fan_in) / 0.1 if (weight_scale and scaled) else 1.0
            out = np.empty(rows * cols, dtype=F32)
            step = 1 << 22

            def work(off):
                u = uniform_stream(seed, min(step, out.size - off), start + off)
                out[off : off + u.size] = bf16((u * scale).astype(F32) if scale != 1.0 else u.astype(F32))

            with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
                list(ex.map(work, range(0, out.size, step)))
            return out.reshape(rows, cols)

        self.embedding = mat(0, vocab, d, d, scaled=False)
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

    def norm_split(self, x):
        """The folded RMSNorm: (bf16(x), r) — a projection of the normed row is (h @ W) * r."""
        x = x.astype(F32)
        return bf16(x), rms_scale_gpu_order(x, self.eps)[0]

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
        h, r = self.norm_split(x)
        q = self.rope((h @ w["wq"]) * r, pos)
        k = self.rope((h @ w["wk"]) * r, pos)
        v = (h @ w["wv"]) * r
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
        h2, r2 = self.norm_split(x)
        g = (h2 @ w["wg"]) * r2
        u = (h2 @ w["wu"]) * r2
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

    def new_dense_kv(self, capacity: int = 256) -> DenseKv:
        return DenseKv(self.layers, self.kv_heads * 128, capacity)

    # -- batched restatement (same per-node semantics, GEMMs over a level) ----
    def norm_rows(self, x):
        x = x.astype(F32)
        r = F32(1.0) / np.sqrt(np.mean(x * x, axis=1, dtype=F32) + F32(self.eps), dtype=F32)
        return bf16(x * r[:, None])

    def norm_split_rows(self, x):
        x = x.astype(F32)
        return bf16(x), rms_scale_gpu_order(x, self.eps)[:, None]

    def rope_rows(self, y, pos):
        ang = np.asarray(pos, dtype=np.float64)[:, None] * self._inv[None, :]
        c, s = np.cos(ang).astype(F32)[:, None, :], np.sin(ang).astype(F32)[:, None, :]
        n = y.shape[0]
        y = y.reshape(n, -1, 128)
        y1, y2 = y[..., :64], y[..., 64:]
        return np.concatenate([y1 * c - y2 * s, y2 * c + y1 * s], axis=2).reshape(n, -1)

    def block_many(self, layer, x, kv: DenseKv, row_lists, append, pos):
        """``block`` for n nodes at once.  Node i attends the stored rows
        ``row_lists[i]`` (in that order) then its own K/V (self last), exactly
        the per-node rule of `model.py:265-271`; with ``append`` the n new K/V
        rows are stored first (rows len(kv)-n .. in node order)."""
        w = self.blocks[layer]
        n = x.shape[0]
        h, r = self.norm_split_rows(x)
        qb = bf16(self.rope_rows((h @ w["wq"]) * r, pos))
        kb = bf16(self.rope_rows((h @ w["wk"]) * r, pos))
        vb = bf16((h @ w["wv"]) * r)
        if append:
            kv.put_many(layer, kb, vb)
        g = self.heads // self.kv_heads
        scale = F32(1.0 / np.sqrt(128.0))
        out = np.empty((n, self.heads * 128), dtype=F32)
        for i in range(n):
            rows = row_lists[i]
            ks = np.concatenate([kv.k_rows(layer, rows), kb[i : i + 1]]).reshape(-1, self.kv_heads, 128)
            vs = np.concatenate([kv.v_rows(layer, rows), vb[i : i + 1]]).reshape(-1, self.kv_heads, 128)
            q = qb[i].reshape(self.kv_heads, g, 128)
            sc = np.einsum("kgd,rkd->kgr", q, ks) * scale
            p = np.exp(sc - sc.max(axis=2, keepdims=True)).astype(F32)
            o = np.einsum("kgr,rkd->kgd", bf16(p), vs) / p.sum(axis=2, dtype=F32)[..., None]
            out[i] = o.reshape(-1)
        x = x + bf16(out) @ w["wo"]
        h2, r2 = self.norm_split_rows(x)
        gg = (h2 @ w["wg"]) * r2
        u = (h2 @ w["wu"]) * r2
        a = bf16((gg / (F32(1.0) + np.exp(-gg))) * u)
        return (x + a @ w["wd"]).astype(F32)

    def causal_block(self, layer, x, kv: DenseKv, pos):
        """Prompt block: row r0+i attends rows [0, r0+i) then self (prefill,
        `pipeline.py:247-254`), computed as one masked attention per KV head."""
        w = self.blocks[layer]
        n = x.shape[0]
        h, r = self.norm_split_rows(x)
        qb = bf16(self.rope_rows((h @ w["wq"]) * r, pos))
        kb = bf16(self.rope_rows((h @ w["wk"]) * r, pos))
        vb = bf16((h @ w["wv"]) * r)
        kv.put_many(layer, kb, vb)
        tot = kv.filled[layer]
        r0 = tot - n
        K = kv.keys(layer).reshape(tot, self.kv_heads, 128)
        V = kv.values(layer).reshape(tot, self.kv_heads, 128)
        g = self.heads // self.kv_heads
        scale = F32(1.0 / np.sqrt(128.0))
        mask = np.arange(tot)[None, :] > (r0 + np.arange(n))[:, None]
        out = np.empty((n, self.heads, 128), dtype=F32)
        q = qb.reshape(n, self.heads, 128)
        for hh in range(self.heads):
            kh = hh // g
            sc = (q[:, hh] @ K[:, kh].T) * scale
            sc[mask] = -np.inf
            p = np.exp(sc - sc.max(axis=1, keepdims=True)).astype(F32)
            out[:, hh] = (bf16(p) @ V[:, kh]) / p.sum(axis=1, dtype=F32)[:, None]
        x = x + bf16(out.reshape(n, -1)) @ w["wo"]
        h2, r2 = self.norm_split_rows(x)
        gg = (h2 @ w["wg"]) * r2
        u = (h2 @ w["wu"]) * r2
        a = bf16((gg / (F32(1.0) + np.exp(-gg))) * u)
        return (x + a @ w["wd"]).astype(F32)

    def prefill_block(self, tokens, kv: DenseKv, start_pos=0, layer_range=None, x_in=None, chunk=512):
        """Causal prompt forward of ``tokens`` (or rows ``x_in``) in chunks."""
        lo, hi = layer_range if layer_range is not None else self.layer_range
        n = len(tokens) if x_in is None else len(x_in)
        outs = []
        for s0 in range(0, n, chunk):
            s1 = min(n, s0 + chunk)
            x = (self.embedding[np.asarray(tokens[s0:s1])].astype(F32) if x_in is None
                 else np.asarray(x_in[s0:s1], dtype=F32))
            pos = np.arange(start_pos + s0, start_pos + s1)
            for p in pos:
                kv.open_row(-1, int(p), True)
            for layer in range(lo, hi):
                x = self.causal_block(layer, x, kv, pos)
            outs.append(x)
        return np.concatenate(outs)

    def forward_level(self, kv: DenseKv, nodes, embeddings=None, layer_range=None, append=True):
        """``forward_tree`` (`model.py:312-349`) for a batch of
        (uid, token, position, ancestors) nodes, none of which is an
        ancestor of another (a tree level): rows = prefix ∪ ancestors, in
        cache order, then self; recompute mode drops same-position rows."""
        lo, hi = layer_range if layer_range is not None else self.layer_range
        rows = []
        for uid, _tok, pos, anc in nodes:
            r = kv.allowed(anc)
            if not append:
                r = [i for i in r if kv.positions[i] != pos]
            rows.append(r)
        x = (self.embedding[np.asarray([nd[1] for nd in nodes])].astype(F32) if embeddings is None
             else np.asarray(embeddings, dtype=F32))
        pos = np.asarray([nd[2] for nd in nodes])
        if append:
            for uid, _tok, p, _anc in nodes:
                kv.open_row(uid, int(p), False)
        for layer in range(lo, hi):
            x = self.block_many(layer, x, kv, rows, append, pos)
        return x
