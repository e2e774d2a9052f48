"""SpecPipe-DB throughput (BASELINE config 5): 13B-shape target, 8 stages on
one GPU, FIFO stream of B synthetic requests, total tree width 64, combined
ragged GPU tick.  Prints one JSON object per batch size.

    python scripts/bench_db.py [--model 13b] [--batches 1,8,32] [--new 24]
"""
import argparse
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def measure_db(model, batch, prompt_len, new_tokens, total_width=64, k=16, stages=8, seed=0, combined=True):
    import paper_2504_04104_b200 as tp

    V = model.cfg.vocab
    reqs = [tp.Request(i, 0, tuple(int(t) for t in np.random.default_rng([seed, i + 1]).integers(0, V, prompt_len)),
                       new_tokens) for i in range(batch)]
    # same-kernel batched greedy decode (one token per request per forward): the
    # references the drafts bind to, and the steady-state greedy comparator
    # (tokens/s of its decode loop, prefill excluded)
    timing = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    refs = dict(enumerate(tp.sequential_decode_batch(model, [list(r.prompt) for r in reqs], new_tokens, timing)))
    torch.cuda.synchronize()
    ref_s = time.perf_counter() - t0
    greedy_tps = batch * new_tokens / timing["decode_s"]
    bcfg = tp.BatchConfig(max_batch=batch, total_width=total_width, k=k, draft=tp.SyntheticDraftConfig(seed=seed),
                          check_isolation_every_tick=False)
    sched = tp.BatchScheduler(model, tp.PipelineConfig(num_stages=stages), bcfg, references=refs, combined=combined)
    for r in reqs:
        sched.submit(r)
    sched.queue.sort(key=lambda r: (r.arrival_tick, r.request_id))
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    sched.tick()  # admission tick: every request prefilled, first tick
    torch.cuda.synchronize()
    admit_s = time.perf_counter() - t_all
    tok0 = sum(len(s.runner.emitted) for s in sched.active)
    ticks = 0
    gc.collect()  # no cyclic-GC pause inside the timed ticks (as timeit)
    gc.disable()
    t1 = time.perf_counter()
    # steady state: the full batch stays active until the first request finishes
    while len(sched.active) == batch and ticks < 10 * new_tokens:
        sched.tick()
        ticks += 1
    torch.cuda.synchronize()
    steady_s = time.perf_counter() - t1
    gc.enable()
    tokens = sum(len(s.runner.emitted) for s in sched.active + sched.finished) - tok0
    metrics = sched.run()
    torch.cuda.synchronize()
    total_s = time.perf_counter() - t_all
    ok = all(s.runner.emitted[: s.request.max_new_tokens] == refs[s.request.request_id] for s in sched.finished)
    return {"batch": batch, "tokens_per_s": round(tokens / steady_s, 2), "steady_ticks": ticks,
            "ms_per_tick": round(steady_s * 1e3 / max(1, ticks), 3), "tokens_per_tick": round(tokens / max(1, ticks), 3),
            "workload_tokens_per_s": round(metrics.tokens / total_s, 2), "admission_s": round(admit_s, 3),
            "lossless": ok, "reference_decode_s": round(ref_s, 2), "combined": combined,
            "batched_greedy_tokens_per_s": round(greedy_tps, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="13b")
    ap.add_argument("--batches", default="1,2,4,8,16,32,64")
    ap.add_argument("--new", type=int, default=24)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--uncombined", action="store_true")
    args = ap.parse_args()
    from bench import model_cfg
    from paper_2504_04104_b200.model import LlamaModel

    torch.cuda.set_device(0)
    model = LlamaModel(model_cfg(args.model), max_nodes=256)
    batches = [int(x) for x in args.batches.split(",")]
    measure_db(model, min(16, max(batches)), args.prompt_len, 8, combined=not args.uncombined)  # untimed warm-up
    for b in batches:
        print(json.dumps(measure_db(model, b, args.prompt_len, args.new, combined=not args.uncombined)), flush=True)


if __name__ == "__main__":
    main()
