"""Step-machine oracle: restatement of one SpecPipe pipeline step (TEST ONLY).

Follows `/root/reference/pkg/src/treepipe/pipeline.py:239-490`
(prefill / step / decode_step) with the tree ops of `tree.py:116-188`
and the frontier expansion of `token_source.py:229-257`, written over a
plain boolean mask and Python uid sets.  It is model-agnostic: any object
with ``embed``/``greedy``/``run_position``/``layers``/``hidden`` works
(``oracle.toy.ToyOracle`` or ``oracle.llama.LlamaOracle``).

Per step it records what the parity tests compare bit-exactly against the
B200 engine: the verified token, hit/miss, every stage's KV keep list in
cache-row space (the reference ``KvCache._restrict`` argument,
`model.py:184`) and the reference wire encoding of the tree.
"""

from __future__ import annotations

import itertools
import struct

import numpy as np

from .toy import OracleKv, forward_nodes


def _exc_named(exc: BaseException, name: str) -> bool:
    return any(c.__name__ == name for c in type(exc).__mro__)


class OTree:
    """BFS tree over a bool ancestor-or-self mask."""

    _uids = itertools.count(10_000_000)

    def __init__(self, tokens, probs, mask, offsets, uids):
        self.tokens, self.probs, self.mask, self.offsets, self.uids = tokens, probs, mask, offsets, uids

    @classmethod
    def root(cls, token):
        return cls([int(token)], [1.0], np.ones((1, 1), bool), [0], [next(cls._uids)])

    @property
    def n(self):
        return len(self.tokens)

    def bounds(self, level):
        lo = self.offsets[level]
        return lo, (self.offsets[level + 1] if level + 1 < len(self.offsets) else self.n)

    def depth(self, i):
        return max(l for l, o in enumerate(self.offsets) if o <= i)

    def grow(self, children):
        n, k = self.n, len(children)
        m = np.zeros((n + k, n + k), bool)
        m[:n, :n] = self.mask
        for j, (p, _, _) in enumerate(children):
            m[n + j, :n] = self.mask[p]
            m[n + j, n + j] = True
        return OTree(self.tokens + [int(c[1]) for c in children], self.probs + [c[2] for c in children],
                     m, self.offsets + [n], self.uids + [next(self._uids) for _ in range(k)])

    def reroot(self, r):
        keep = np.flatnonzero(self.mask[:, r])
        shift = self.depth(r)
        depths = [self.depth(int(i)) - shift for i in keep]
        offsets = [depths.index(d) for d in range(depths[-1] + 1)]
        probs = [self.probs[int(i)] for i in keep]
        probs[0] = 1.0
        return OTree([self.tokens[int(i)] for i in keep], probs, self.mask[np.ix_(keep, keep)].copy(),
                     offsets, [self.uids[int(i)] for i in keep])

    def encode(self) -> bytes:
        n = self.n
        return (struct.pack("<II", n, len(self.offsets))
                + np.asarray(self.tokens, "<u4").tobytes() + np.asarray(self.probs, "<f8").tobytes()
                + np.asarray(self.offsets, "<u4").tobytes()
                + np.packbits(self.mask, axis=1, bitorder="little").tobytes())


def oracle_expand(tree: OTree, w: int, k: int, draft, context, step: int):
    lo, hi = tree.bounds(len(tree.offsets) - 1)
    pool = []
    for node in range(lo, hi):
        path = np.flatnonzero(tree.mask[node])
        ctx = tuple(context) + tuple(tree.tokens[int(j)] for j in path[1:])
        cum = float(np.prod(np.asarray(tree.probs)[tree.mask[node]]))
        for tok, p in draft.propose(ctx, k, step=step, frontier_node=node):
            pool.append((p * cum, node, tok, p))
    pool.sort(key=lambda c: (-c[0], c[1], c[2]))
    return [(nd, t, p) for _, nd, t, p in sorted(pool[:w], key=lambda c: (c[1], -c[3], c[2]))]


def split_even(layers: int, stages: int):
    base, rem = divmod(layers, stages)
    out, lo = [], 0
    for i in range(stages):
        hi = lo + base + (1 if i < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


class OracleRunner:
    def __init__(self, model, num_stages, w, k, draft=None, splits=None, new_kv=None):
        self.model, self.w, self.k, self.draft = model, w, k, draft
        self.splits = splits or split_even(model.layers, num_stages)
        new_kv = new_kv or (lambda: OracleKv(model.layers, model.hidden))
        self.stages = [{"kv": new_kv(), "res": None, "out": None, "range": r} for r in self.splits]
        self.tree = None
        self.verified, self.emitted = [], []
        self.pos, self.verified_uids = {}, set()
        self.hits = self.misses = self.steps = 0
        self.log = []

    def _payload(self, level, cached=False):
        lo, hi = self.tree.bounds(level)
        t = self.tree
        return {"uids": [t.uids[i] for i in range(lo, hi)],
                "tokens": [t.tokens[i] for i in range(lo, hi)],
                "pos": [self.pos[t.uids[i]] for i in range(lo, hi)],
                "anc": [frozenset(t.uids[int(j)] for j in np.flatnonzero(t.mask[i])) for i in range(lo, hi)],
                "emb": None, "cached": cached}

    def prefill(self, prompt, batched=False):
        """Prompt through every stage (`pipeline.py:239-268`): one position at a
        time as the reference, or — ``batched`` (Llama oracle, DenseKv caches) —
        as one causal block per stage (same semantics, GEMMs; used to set up the
        CPU timing arm, whose timed region is the decode steps)."""
        if batched:
            x = None
            for st in self.stages:
                x = self.model.prefill_block(prompt, st["kv"], 0, st["range"], x_in=x)
        else:
            for p, tok in enumerate(prompt):
                x = self.model.embed(tok, p)
                for st in self.stages:
                    x = self.model.run_position(x, st["kv"], list(range(len(st["kv"]))), st["range"],
                                                True, -1, p, True)
        self.verified = list(prompt)
        self.tree = OTree.root(prompt[-1])
        self.pos[self.tree.uids[0]] = len(prompt) - 1
        self.verified_uids.add(self.tree.uids[0])
        self.stages[0]["res"] = self._payload(0, cached=True)

    def step(self, children):
        self.steps += 1
        stalled = not children
        levels_before = len(self.tree.offsets)
        if not stalled:
            self.tree = self.tree.grow(children)
            lo, hi = self.tree.bounds(len(self.tree.offsets) - 1)
            for i, (par, _, _) in enumerate(children):
                self.pos[self.tree.uids[lo + i]] = self.pos[self.tree.uids[par]] + 1
        for st in self.stages:
            r = st["res"]
            st["out"] = None if r is None else forward_nodes(
                self.model, st["kv"], list(zip(r["uids"], r["tokens"], r["pos"], r["anc"])),
                r["emb"], st["range"], append=not r["cached"])
        last = self.stages[-1]
        rec = {"token": None, "hit": False, "keeps": None, "outs": [s["out"] for s in self.stages]}
        tok, keep_uids = None, None
        if last["res"] is not None:
            assert last["res"]["uids"] == [self.tree.uids[0]]
            tok = self.model.greedy(last["out"][0])
            self.verified.append(tok)
            self.emitted.append(tok)
            child = None
            if len(self.tree.offsets) >= 2:
                lo, hi = self.tree.bounds(1)
                child = next((i for i in range(lo, hi) if self.tree.tokens[i] == tok), None)
            keeps = []
            if child is not None:
                self.hits += 1
                chain = {self.tree.uids[int(j)] for j in np.flatnonzero(self.tree.mask[child])}
                new = self.tree.reroot(child)
                keep_uids = set(new.uids)
                self.verified_uids |= chain
                for st in self.stages:
                    st["kv"].promote(chain)
                    rows = st["kv"].keep_rows(keep_uids)
                    keeps.append(rows)
                    st["kv"].restrict(rows)
                self.tree = new
            else:
                self.misses += 1
                root = self.tree.uids[0]
                self.verified_uids.add(root)
                for st in self.stages:
                    st["kv"].promote({root})
                    rows = [i for i, p in enumerate(st["kv"].prefix) if p]
                    keeps.append(rows)
                    st["kv"].restrict(rows)
                    st["res"] = st["out"] = None
                self.tree = OTree.root(tok)
                self.pos[self.tree.uids[0]] = len(self.verified) - 1
                self.verified_uids.add(self.tree.uids[0])
            rec.update(token=tok, hit=child is not None, keeps=keeps)
        outgoing = []
        for st in self.stages:
            r = st["res"]
            if r is None or st["out"] is None:
                outgoing.append(None)
                continue
            idx = list(range(len(r["uids"]))) if keep_uids is None else \
                [i for i, u in enumerate(r["uids"]) if u in keep_uids]
            outgoing.append(None if not idx else {
                "uids": [r["uids"][i] for i in idx], "tokens": [r["tokens"][i] for i in idx],
                "pos": [r["pos"][i] for i in idx], "anc": [r["anc"][i] for i in idx],
                "emb": st["out"][idx], "cached": r["cached"]})
        if tok is None:
            new_level = None if stalled else self._payload(len(self.tree.offsets) - 1)
        elif keep_uids is not None:
            if not stalled and len(self.tree.offsets) == levels_before:
                new_level = self._payload(len(self.tree.offsets) - 1)
            else:
                lo, hi = self.tree.bounds(len(self.tree.offsets) - 1)
                self.tree = self.tree.grow([(lo, tok, 1.0)])
                self.pos[self.tree.uids[-1]] = self.pos[self.tree.uids[lo]] + 1
                new_level = self._payload(len(self.tree.offsets) - 1)
        else:
            new_level = self._payload(0, cached=False)
        for i in range(len(self.stages) - 1, 0, -1):
            self.stages[i]["res"] = outgoing[i - 1]
        self.stages[0]["res"] = new_level
        for st in self.stages:
            st["out"] = None
        rec["tree"] = self.tree.encode()
        self.log.append(rec)
        return rec

    def decode_step(self):
        try:
            children = oracle_expand(self.tree, self.w, self.k, self.draft, self.verified, self.steps + 1)
        except Exception as exc:  # noqa: BLE001 - mirror reference stall handling
            if _exc_named(exc, "DraftExhausted") or not _exc_named(exc, "SourceUnavailable"):
                raise
            children = None
        return self.step(children)

    def run(self, prompt, max_tokens):
        self.prefill(prompt)
        while len(self.emitted) < max_tokens:
            try:
                self.decode_step()
            except Exception as exc:  # noqa: BLE001
                if _exc_named(exc, "DraftExhausted"):
                    break
                raise
        return list(self.emitted)
