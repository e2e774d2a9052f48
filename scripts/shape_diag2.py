"""One token through one 7B-shape layer: GPU kernels vs float32 oracle vs a float64 torch restatement."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, prefill_rows
from oracle.llama import LlamaOracle, bf16

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64); d = a - b
    return float(np.abs(d).max() / np.abs(b).max()), float(np.sqrt((d * d).mean() / (b * b).mean()))

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
cfg = {"7b": LlamaConfig.llama2_7b(), "tiny": LlamaConfig(vocab=512, hidden=256, layers=2, heads=2, kv_heads=1, ffn=512)}[name]
m = LlamaModel(cfg, max_nodes=64, layer_range=(0, 1), with_embed=True, with_head=False)
o = LlamaOracle(cfg.vocab, cfg.hidden, cfg.layers, cfg.heads, cfg.kv_heads, cfg.ffn, layer_range=(0, 1), with_head=False)
d, q, kv, f = cfg.hidden, cfg.heads * 128, cfg.kv_heads * 128, cfg.ffn
def W(which, shape):
    u = m.read_tensor(which, 0).view(np.uint16)
    return torch.from_numpy((u.astype(np.uint32) << 16).view(np.float32).reshape(shape)).double().cuda()
Wqkv = W(1, (q + 2 * kv, d)); Wo = W(4, (d, q)); Wgu = W(5, (2 * f // 128, 2, 64, d)); Wd = W(7, (d, f))
Wg = Wgu[:, 0].reshape(f, d); Wu = Wgu[:, 1].reshape(f, d)
print("weights eq oracle:", np.array_equal(Wo.cpu().numpy(), o.blocks[0]["wo"].T), np.array_equal(Wd.cpu().numpy(), o.blocks[0]["wd"].T))
tok = 123
c = KvCache(cfg.layers, cfg.hidden, capacity=8).bind(m, (0, 1))
xg = prefill_rows(m, c, [tok], layer_range=(0, 1))[0].cpu().numpy()
kvo = o.new_dense_kv(8)
xo = o.prefill_block([tok], kvo)[0]
def bfr(t):
    return t.float().to(torch.bfloat16).double()
x0 = torch.from_numpy(o.embedding[tok].astype(np.float64)).cuda()
def norm(x):
    return bfr(x * torch.rsqrt((x * x).mean() + 1e-5))
h = norm(x0)
v = bfr(Wqkv[q + kv:] @ h)
o1 = x0 + Wo @ v
h2 = norm(o1)
g = Wg @ h2; u = Wu @ h2
a = bfr(g / (1 + torch.exp(-g)) * u)
x1 = (o1 + Wd @ a).cpu().numpy()
print("gpu vs f64", rel(xg, x1), "oracle vs f64", rel(xo, x1), "gpu vs oracle", rel(xg, xo))
# oracle intermediates
w = o.blocks[0]
ho = o.norm(o.embedding[tok].astype(np.float32))
vo = bf16(ho @ w["wv"])
print("v oracle vs f64", rel(vo, v.cpu().numpy()))
o1o = o.embedding[tok].astype(np.float32) + vo @ w["wo"]
print("o1 oracle vs f64", rel(o1o, o1.cpu().numpy()))
