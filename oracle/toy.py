"""Toy-arch oracle: numpy float64 restatement of the reference decoder (TEST ONLY).

Follows `/root/reference/pkg/src/treepipe/model.py`:
  * weights from the LCG stream in the order embedding, then per layer
    Wq, Wk, Wv, Wo (d x d), W1 (d x 2d), W2 (2d x d)        (`model.py:207-235`)
  * embed = E[token] + interleaved sinusoid(pos)             (`model.py:89-102,239-240`)
  * pre-LN block, parameter-free LN (population var, eps 1e-6 in sqrt),
    single-head attention over gathered rows + self (self last),
    ReLU FFN                                                 (`model.py:83-86,250-280`)
  * tied head, greedy = first argmax                         (`model.py:242-248`)
  * KV rows: prefix rows are permanent, speculative rows carry a uid;
    rows_for / promote / prune / drop_speculative            (`model.py:105-204`)
  * forward_tree: per node in BFS order, attention restricted to
    prefix ∪ ancestors; recompute mode drops same-position rows
                                                             (`model.py:312-349`)
The float ops are issued in the same order as the reference (one position
at a time, numpy matvecs), so results are bit-identical in this image.
"""

from __future__ import annotations

import numpy as np

from .lcg import uniform_stream

EPS = 1e-6


class ToyOracle:
    def __init__(self, vocab: int, hidden: int, layers: int, seed: int):
        if vocab < 16 or hidden % 2 or layers < 2:
            raise ValueError("invalid toy config")
        self.vocab, self.hidden, self.layers, self.seed = vocab, hidden, layers, seed
        d, f = hidden, 2 * hidden
        sizes = [vocab * d] + [4 * d * d + 2 * d * f] * layers
        stream = uniform_stream(seed, sum(sizes))
        cursor = [0]

        def take(r, c):
            blk = stream[cursor[0] : cursor[0] + r * c].reshape(r, c)
            cursor[0] += r * c
            return blk

        self.embedding = take(vocab, d)
        self.blocks = []
        for _ in range(layers):
            self.blocks.append(
                {name: take(*shape) for name, shape in
                 (("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)), ("wo", (d, d)),
                  ("w1", (d, f)), ("w2", (f, d)))}
            )
        half = d // 2
        self._freqs = np.exp(-np.log(10000.0) * np.arange(half) / half)

    # -- pieces ---------------------------------------------------------------
    @staticmethod
    def norm(x: np.ndarray) -> np.ndarray:
        return (x - x.mean()) / np.sqrt(x.var() + EPS)

    def position(self, pos: int) -> np.ndarray:
        ang = pos * self._freqs
        enc = np.empty(self.hidden)
        enc[0::2] = np.sin(ang)
        enc[1::2] = np.cos(ang)
        return enc

    def embed(self, token: int, pos: int) -> np.ndarray:
        return self.embedding[token] + self.position(pos)

    def logits(self, x: np.ndarray) -> np.ndarray:
        return self.embedding @ self.norm(x)

    def greedy(self, x: np.ndarray) -> int:
        return int(np.argmax(self.logits(x)))

    def block(self, layer: int, x, kv: "OracleKv", rows, append: bool):
        w = self.blocks[layer]
        h = self.norm(x)
        q, k, v = h @ w["wq"], h @ w["wk"], h @ w["wv"]
        if append:
            kv.put(layer, k, v)
        ks = np.concatenate([kv.k_rows(layer, rows), k[None, :]])
        vs = np.concatenate([kv.v_rows(layer, rows), v[None, :]])
        s = ks @ q / np.sqrt(self.hidden)
        s -= s.max()
        p = np.exp(s)
        p /= p.sum()
        x = x + (p @ vs) @ w["wo"]
        h2 = self.norm(x)
        return x + np.maximum(h2 @ w["w1"], 0.0) @ w["w2"]

    def run_position(self, x, kv, rows, layer_range=None, append=True, uid=-1, pos=0, prefix=False):
        lo, hi = layer_range if layer_range is not None else (0, self.layers)
        if append:
            kv.open_row(uid, pos, prefix)
        for layer in range(lo, hi):
            x = self.block(layer, x, kv, rows, append)
        return x


class OracleKv:
    """Row store with the reference KvCache semantics (per-layer K/V rows,
    shared uid / position / prefix metadata)."""

    def __init__(self, layers: int, hidden: int):
        self.hidden = hidden
        self.k = [[] for _ in range(layers)]
        self.v = [[] for _ in range(layers)]
        self.uids: list[int] = []
        self.positions: list[int] = []
        self.prefix: list[bool] = []

    def __len__(self):
        return len(self.uids)

    def open_row(self, uid, pos, prefix):
        self.uids.append(uid)
        self.positions.append(pos)
        self.prefix.append(prefix)

    def put(self, layer, k, v):
        self.k[layer].append(k)
        self.v[layer].append(v)

    def _rows(self, store, rows):
        if not rows:
            return np.empty((0, self.hidden))
        return np.stack([store[i] for i in rows])

    def k_rows(self, layer, rows):
        return self._rows(self.k[layer], rows)

    def v_rows(self, layer, rows):
        return self._rows(self.v[layer], rows)

    def keys(self, layer) -> np.ndarray:
        return self._rows(self.k[layer], list(range(len(self.k[layer]))))

    def values(self, layer) -> np.ndarray:
        return self._rows(self.v[layer], list(range(len(self.v[layer]))))

    def allowed(self, ancestors) -> list[int]:
        return [i for i in range(len(self.uids)) if self.prefix[i] or self.uids[i] in ancestors]

    def spec_uids(self) -> set[int]:
        return {u for u, p in zip(self.uids, self.prefix) if not p}

    def promote(self, uids) -> None:
        for i, u in enumerate(self.uids):
            if u in uids:
                self.prefix[i] = True
                self.uids[i] = -1

    def keep_rows(self, keep_uids) -> list[int]:
        return [i for i in range(len(self.uids)) if self.prefix[i] or self.uids[i] in keep_uids]

    def restrict(self, keep: list[int]) -> None:
        for layer in range(len(self.k)):
            if self.k[layer]:
                self.k[layer] = [self.k[layer][i] for i in keep]
                self.v[layer] = [self.v[layer][i] for i in keep]
        self.uids = [self.uids[i] for i in keep]
        self.positions = [self.positions[i] for i in keep]
        self.prefix = [self.prefix[i] for i in keep]


def forward_nodes(model, kv: OracleKv, nodes, embeddings=None, layer_range=None, append=True):
    """Reference ``forward_tree`` (`model.py:312-349`) for (uid, token, pos, ancestors)."""
    outs = []
    for idx, (uid, token, pos, anc) in enumerate(nodes):
        x = model.embed(token, pos) if embeddings is None else embeddings[idx]
        rows = kv.allowed(anc)
        if not append:
            rows = [i for i in rows if kv.positions[i] != pos]
        outs.append(model.run_position(x, kv, rows, layer_range, append, uid, pos))
    return np.stack(outs)


def greedy_continuation(model, prompt, steps):
    """Reference ``sequential_decode`` (`model.py:364-385`)."""
    kv = OracleKv(model.layers, model.hidden)
    x = None
    for pos, tok in enumerate(prompt):
        x = model.run_position(model.embed(tok, pos), kv, list(range(len(kv))), pos=pos, prefix=True)
    out = []
    pos = len(prompt)
    for _ in range(steps):
        tok = model.greedy(x)
        out.append(tok)
        x = model.run_position(model.embed(tok, pos), kv, list(range(len(kv))), pos=pos, prefix=True)
        pos += 1
    return out
