"""K1 run-kernel timeline from the globaltimer trace (library built with
TP_NVCC_EXTRA=-DTP_ATTN_TRACE).  One grouped phase-1 forward of the 7B bench
shape (7 stages, mean node counts, 512 prefix); the trace holds the last
attention launch (last layer slot).

    TP_NVCC_EXTRA=-DTP_ATTN_TRACE python -m paper_2504_04104_b200.build && python scripts/attn_trace.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from bench import model_cfg  # noqa: E402
from paper_2504_04104_b200 import _lib  # noqa: E402
from paper_2504_04104_b200.model import LlamaModel, forward_members  # noqa: E402
from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner  # noqa: E402

mask = int(os.environ.get("MASK", "0"))
prefix = int(os.environ.get("PREFIX", "512"))
cfg = model_cfg("7b")
m = LlamaModel(cfg, max_nodes=64)
ns = [int(x) for x in os.environ.get("NS", "45,35,29,23,17,11,3").split(",")]
depth = 12
prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab, prefix + depth)]
r = PipelineRunner(m, PipelineConfig(num_stages=8), tp.BeamConfig(w=64, k=16), None, collect_trace=False,
                   kv_capacity=max(2048, prefix + 256))
r.prefill(prompt)
rng = np.random.default_rng(2)
items = []
for s, n in zip(r.stages, ns):
    d = rng.integers(0, depth, n)
    pre = np.full(n, prefix, dtype=np.int32)
    bits = ((np.uint64(1) << d.astype(np.uint64)) - np.uint64(1)).reshape(n, 1).astype(np.uint64)
    x = torch.randn(n, cfg.hidden, device="cuda") * 0.5  # fp32 residual-stream rows
    items.append((s.kv, m, x, None, (prefix + d).tolist(), s.layer_range, False, list(range(n)), False,
                  (pre, prefix, 1, bits)))
lib = _lib.lib()
members = [[it] for it in items]
_lib.check(lib.tp_debug_attn_knob(3, mask))
for _ in range(3):
    forward_members(members)
torch.cuda.synchronize()
buf = torch.zeros(296 * 8 * 1024, dtype=torch.int64, device="cuda")
_lib.check(lib.tp_debug_attn_trace(buf.data_ptr()))
forward_members(members)
torch.cuda.synchronize()
_lib.check(lib.tp_debug_attn_trace(None))
_lib.check(lib.tp_debug_attn_knob(3, 0))
tr = buf.cpu().numpy().view(np.uint64).reshape(296, 8, 1024)
tag = (tr >> np.uint64(56)).astype(np.int64)
arg = ((tr >> np.uint64(40)) & np.uint64(0xFFFF)).astype(np.int64)
tim = (tr & np.uint64(0xFFFFFFFFFF)).astype(np.int64)
live = tr[:, 0, 0] != 0
start = np.where(live, tim[:, 0, 0], np.iinfo(np.int64).max)
t0 = start[live].min()
ev = {}
for c in np.nonzero(live)[0]:
    for role in range(4):
        for i in range(1024):
            if tr[c, role, i] == 0 or tim[c, role, i] < start[c]:
                break
            ev.setdefault(tag[c, role, i], []).append((c, arg[c, role, i], tim[c, role, i] - t0))
end = {}
for k, lst in ev.items():
    for c, a, t in lst:
        end[c] = max(end.get(c, 0), t)
print("CTAs traced", int(live.sum()), "start (us rel): med/max", np.median(start[live] - t0) / 1e3, (start[live].max() - t0) / 1e3)
print("CTA end   (us rel): min/med/max", min(end.values()) / 1e3, np.median(list(end.values())) / 1e3,
      max(end.values()) / 1e3)
key = {}
for k in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13):
    for c, a, t in ev.get(k, []):
        key[(k, c, a)] = t
def lat(a_tag, b_tag, shift=0):
    d = [key[(b_tag, c, a + shift)] - t for (k, c, a), t in key.items() if k == a_tag and (b_tag, c, a + shift) in key]
    return (np.median(d) / 1e3, np.mean(d) / 1e3, len(d)) if d else None
print("producer issue -> S issued (kv wait)      ", lat(4, 5))
print("S issued -> softmax sees S                ", lat(5, 1))
print("softmax sees S -> P arrive (softmax time) ", lat(1, 2))
print("  S seen -> tmem ld done                ", lat(1, 8))
print("  ld done -> max exchanged               ", lat(8, 9))
print("  exchanged -> exp/pack done             ", lat(9, 10))
print("  exp done -> before P store (rescale/wait)", lat(10, 11))
print("  before P store -> P arrive             ", lat(11, 2))
print("P arrive -> PV issued                     ", lat(2, 6))
print("softmax S(g) -> S(g+1)  (chunk period)    ", lat(1, 1, 1))
print("producer issue(g) -> issue(g+1)           ", lat(4, 4, 1))
print("chunks per CTA: ", np.bincount([c for c, a, t in ev.get(1, [])], minlength=296).mean())
print("tasks per CTA:  ", np.bincount([c for c, a, t in ev.get(7, [])], minlength=296).mean() if 7 in ev else None)
# per-chunk-index arrival of S at the softmax (tag 1) and P arrive (tag 2), median over CTAs
for g in range(8):
    s1 = [t for (k, c, a), t in key.items() if k == 1 and a == g]
    s2 = [t for (k, c, a), t in key.items() if k == 2 and a == g]
    if s1:
        print(f"chunk {g}: S seen med {np.median(s1) / 1e3:6.2f} us  P done med {np.median(s2) / 1e3:6.2f} us  ({len(s1)} CTAs)")
for g in range(8):
    row = []
    for k_, name in ((4, "kv issued"), (5, "S issued"), (1, "S seen"), (2, "P done"), (6, "PV issued")):
        v = [t for (k, c, a), t in key.items() if k == k_ and a == g]
        row.append(f"{name} {np.median(v) / 1e3:6.2f}" if v else f"{name}   -   ")
    print(f"chunk {g}: " + " | ".join(row))
for it in range(3):
    v = [t for (k, c, a), t in key.items() if k == 7 and a == it]
    if v:
        print(f"task it {it}: Q staged med {np.median(v) / 1e3:6.2f} us ({len(v)} CTAs)")
print("task end: last P done -> PV done", lat(2, 3), " PV done -> O stored", lat(3, 12), " O stored -> state stored", lat(12, 13))
