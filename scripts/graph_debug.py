import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2504_04104_b200 as tp
cfg = tp.LlamaConfig(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
m = tp.LlamaModel(cfg, max_nodes=64)
print(tp.sequential_decode(m, [1, 2, 3, 4, 5], 6))
