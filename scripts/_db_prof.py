import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2504_04104_b200 as tp
from bench import model_cfg
from paper_2504_04104_b200.model import LlamaModel
m = LlamaModel(model_cfg("13b"), max_nodes=64)
B, new = 16, 24
V = m.cfg.vocab
reqs = [tp.Request(i, 0, tuple(int(t) for t in np.random.default_rng([0, i + 1]).integers(0, V, 512)), new) for i in range(B)]
refs = dict(enumerate(tp.sequential_decode_batch(m, [list(r.prompt) for r in reqs], new)))
bcfg = tp.BatchConfig(max_batch=B, total_width=64, k=16, draft=tp.SyntheticDraftConfig(seed=0), check_isolation_every_tick=False)
sched = tp.BatchScheduler(m, tp.PipelineConfig(num_stages=8), bcfg, references=refs)
for r in reqs: sched.submit(r)
sched.queue.sort(key=lambda r: (r.arrival_tick, r.request_id))
sched.tick(); sched.tick(); sched.tick()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
for _ in range(20): sched.tick()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 20
pr.disable()
print(f"ms/tick {dt*1e3:.2f}")
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25); st.sort_stats("cumulative").print_stats(25)
