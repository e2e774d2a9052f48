"""K2 phases inside a real launch chain: one lone 4-layer stage forward of the 7B
bench (stage 1 of 8, n nodes, 512 prefix + tree ancestors) with the library built
with -DTP_GEMM_TRACE (`bash scripts/build_variant.sh trace -DTP_GEMM_TRACE`, run
with TP_LIB_VARIANT=trace).  Per GEMM launch, us from the first CTA start of the
forward: CTA start (min/med/max), first MMA, last MMA, CTA end (med/max), and the
gap from the previous GEMM launch's last CTA end (attention sits between qkv and o).

    TP_LIB_VARIANT=trace python scripts/gemm_chain_trace.py [--n 45]
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=45)
ap.add_argument("--prefix", type=int, default=512)
ap.add_argument("--group", default="", help="grouped forward instead: node counts of stages 1..7, e.g. 45,35,29,23,17,11,3")
args = ap.parse_args()
cfg = model_cfg("7b")
m = LlamaModel(cfg, max_nodes=64)
depth = 12
prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab, args.prefix + depth)]
r = PipelineRunner(m, PipelineConfig(num_stages=8), tp.BeamConfig(w=64, k=16), None, collect_trace=False,
                   kv_capacity=2048)
r.prefill(prompt)
rng = np.random.default_rng(2)
s, n = r.stages[0], args.n
d = rng.integers(0, depth, n)
pre = np.full(n, args.prefix, dtype=np.int32)
bits = ((np.uint64(1) << d.astype(np.uint64)) - np.uint64(1)).reshape(n, 1).astype(np.uint64)
x = torch.randn(n, cfg.hidden, device="cuda") * 0.5
members = [[(s.kv, m, x, None, (args.prefix + d).tolist(), s.layer_range, False, list(range(n)), False,
             (pre, args.prefix, 1, bits))]]
if args.group:  # one member per stage, as the bench's phase-1 grouped launch
    members = []
    for st, ng in zip(r.stages, [int(v) for v in args.group.split(",")]):
        dg = rng.integers(0, depth, ng)
        bg = ((np.uint64(1) << dg.astype(np.uint64)) - np.uint64(1)).reshape(ng, 1).astype(np.uint64)
        members.append([(st.kv, m, torch.randn(ng, cfg.hidden, device="cuda") * 0.5, None, (args.prefix + dg).tolist(),
                         st.layer_range, False, list(range(ng)), False, (np.full(ng, args.prefix, dtype=np.int32),
                                                                         args.prefix, 1, bg))])
lib = _lib.lib()
for _ in range(5):
    forward_members(members)
torch.cuda.synchronize()
buf = torch.zeros(64 * 148 * 32, dtype=torch.int64, device="cuda")
_lib.check(lib.tp_debug_gemm_trace(0, buf.data_ptr()))
torch.cuda.profiler.start()  # ncu --profile-from-start off captures this forward only
forward_members(members)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
_lib.check(lib.tp_debug_gemm_trace(0, None))
if not (buf != 0).any():
    print("no trace (library built without -DTP_GEMM_TRACE)")
    sys.exit(0)
t = buf.view(64, 148, 32)[:, :, :21].cpu().numpy().astype(np.float64)
live = [i for i in range(64) if (t[i, :, 0] > 0).any()]
t0 = t[live[0], :, 0][t[live[0], :, 0] > 0].min()
ops = ["qkv", "o", "gu", "down"]
prev_end = None
tot = {}
for j, i in enumerate(live):
    a = t[i]
    ok = a[:, 0] > 0
    rel = (a[ok] - t0) / 1e3
    st, mf, ml, en = rel[:, 0], rel[:, 2], rel[:, 3], rel[:, 8]
    gap = st.min() - prev_end if prev_end is not None else 0.0
    op = ops[j % 4]
    tot.setdefault(op, []).append((en.max() - st.min(), gap, en.max() - ml.max()))
    print(f"L{j // 4} {op:4s} start {st.min():7.1f}/{np.median(st):7.1f}/{st.max():7.1f}  mma {np.median(mf):7.1f}"
          f" .. {np.median(ml):7.1f}/{ml.max():7.1f}  end {np.median(en):7.1f}/{en.max():7.1f}  "
          f"(span {en.max() - st.min():5.1f}, gap before {gap:5.1f}, tail after last MMA {en.max() - ml.max():4.1f})")
    prev_end = en.max()
for op, v in tot.items():
    v = np.array(v)
    print(f"{op:4s} mean span {v[:, 0].mean():5.1f} us, gap before {v[:, 1].mean():5.1f}, tail {v[:, 2].mean():4.1f}")
if os.environ.get("DETAIL"):  # the latest-ending CTAs of one launch, all stamps relative to its first start
    i = live[int(os.environ["DETAIL"])]
    a = t[i]
    ok = np.nonzero(a[:, 0] > 0)[0]
    s0 = a[ok, 0].min()
    names = ["start", "pdl", "mma0", "mmaN", "drain", "spin0", "spin1", "red", "end", "sole0", "sole1", "part0",
             "part1", "rsc", "stg0", "app0", "bar_init", "tmem", "sync", "tmap_pf", "w_issued"]
    for c in ok[np.argsort(-a[ok, 8])][:12]:
        print(f"cta {c:3d}: " + " ".join(f"{nm} {(a[c, k] - s0) / 1e3:5.1f}" if a[c, k] > 0 else f"{nm}   -  "
                                         for k, nm in enumerate(names)))
    med = np.nanmedian(np.where(a[ok] > 0, a[ok] - s0, np.nan) / 1e3, axis=0)
    print("median : " + " ".join(f"{nm} {med[k]:5.1f}" for k, nm in enumerate(names)))
if os.environ.get("PROLOGUE"):  # per-CTA prologue, us from each CTA's own start (median / p90 over CTAs and launches)
    cols = [("bar_init", 16), ("tmem", 17), ("sync", 18), ("tmap_pf", 19), ("w_issued", 20), ("pdl", 1), ("mma0", 2)]
    for j, op in enumerate(ops):
        rel = {nm: [] for nm, _ in cols}
        for i in live[j::4]:
            a = t[i]
            ok = (a[:, 0] > 0)
            for nm, k in cols:
                v = a[ok, k] - a[ok, 0]
                rel[nm] += list(v[a[ok, k] > 0] / 1e3)
        print(f"{op:4s} " + "  ".join(f"{nm} {np.median(v):4.2f}/{np.percentile(v, 90):4.2f}" for nm, v in rel.items() if v))
