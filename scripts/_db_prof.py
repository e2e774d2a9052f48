import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from scripts.bench_db import measure_db
from bench import model_cfg
from paper_2504_04104_b200.model import LlamaModel
m = LlamaModel(model_cfg("13b"), max_nodes=64)
print(measure_db(m, 1, 512, 24))
pr = cProfile.Profile(); pr.enable()
print(measure_db(m, 1, 512, 24))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
