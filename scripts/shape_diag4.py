"""Per-kernel bisection at a Llama shape: GPU intermediates (tp_debug_dump) vs
float64 recomputation from the GPU's own previous intermediate."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_04104_b200 import _lib
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, prefill_rows

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64); d = a - b
    return "max %.2e rms %.2e" % (float(np.abs(d).max() / np.abs(b).max()), float(np.sqrt((d * d).mean() / (b * b).mean())))

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = {"7b": LlamaConfig.llama2_7b(), "tiny": LlamaConfig(vocab=512, hidden=256, layers=2, heads=2, kv_heads=2, ffn=512)}[name]
m = LlamaModel(cfg, max_nodes=64, layer_range=(0, 1), with_embed=True, with_head=False)
d, q, kv, f = cfg.hidden, cfg.heads * 128, cfg.kv_heads * 128, cfg.ffn
def W(which, shape):
    u = m.read_tensor(which, 0).view(np.uint16)
    return torch.from_numpy((u.astype(np.uint32) << 16).view(np.float32).reshape(shape)).double().cuda()
Wqkv = W(1, (q + 2 * kv, d)); Wo = W(4, (d, q)); Wgu = W(5, (2 * f // 128, 2, 64, d)); Wd = W(7, (d, f))
Wg = Wgu[:, 0].reshape(f, d); Wu = Wgu[:, 1].reshape(f, d)
emb = W(0, (cfg.vocab, d))
toks = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab, P)]
n = min(P, 64)
buf = torch.zeros(n * (q * 2 + d * 4 + d * 2 + f * 2 + d * 4), dtype=torch.uint8, device="cuda")
c = KvCache(cfg.layers, cfg.hidden, capacity=P + 8).bind(m, (0, 1))
if P > 64:
    prefill_rows(m, c, toks[:-64], layer_range=(0, 1))
_lib.check(_lib.lib().tp_debug_dump(buf.data_ptr()))
x1 = prefill_rows(m, c, toks[-n:], layer_range=(0, 1)).double()
torch.cuda.synchronize()
o = 0
def take(nbytes, dt, shape):
    global o
    t = buf[o:o + nbytes].view(dt).reshape(shape); o += nbytes
    return t.double() if dt != torch.bfloat16 else t.float().double()
Xo = take(n * q * 2, torch.bfloat16, (n, q))
xo = take(n * d * 4, torch.float32, (n, d))
Xd = take(n * d * 2, torch.bfloat16, (n, d))
Xf = take(n * f * 2, torch.bfloat16, (n, f))
xd = take(n * d * 4, torch.float32, (n, d))
def bfr(t):
    return t.float().to(torch.bfloat16).double()
x0 = emb[toks[-n:]]
print("final x == dump", torch.equal(xd, x1))
print("o-proj: x0 + Xo@Wo^T vs gpu", rel(xo.cpu(), (x0 + Xo @ Wo.t()).cpu()))
nrm = bfr(xo * torch.rsqrt((xo * xo).mean(dim=1, keepdim=True) + cfg.norm_eps))
print("rmsnorm vs f64 of gpu x", rel(Xd.cpu(), nrm.cpu()), "bitwise frac", float((Xd == nrm).double().mean()))
g = Xd @ Wg.t(); u = Xd @ Wu.t()
a = bfr(g / (1 + torch.exp(-g)) * u)
print("swiglu vs f64", rel(Xf.cpu(), a.cpu()), "bitwise frac", float((Xf == a).double().mean()))
print("down: xo + Xf@Wd^T vs gpu", rel(xd.cpu(), (xo + Xf @ Wd.t()).cpu()))
if P == 1:
    h = bfr(x0 * torch.rsqrt((x0 * x0).mean(dim=1, keepdim=True) + cfg.norm_eps))
    v = bfr(h @ Wqkv[q + kv:].t())
    print("attn out (single token = v) vs f64", rel(Xo.cpu(), v.repeat(1, q // kv).cpu()))
if P == 1:
    # whole chain in float64 from x0 (same bf16 rounding points), vs each GPU intermediate
    o1 = x0 + v.repeat(1, q // kv) @ Wo.t()
    h2 = bfr(o1 * torch.rsqrt((o1 * o1).mean(dim=1, keepdim=True) + cfg.norm_eps))
    g2 = h2 @ Wg.t(); u2 = h2 @ Wu.t()
    a2 = bfr(g2 / (1 + torch.exp(-g2)) * u2)
    x2 = o1 + a2 @ Wd.t()
    for tag, gpu, ref in (("o1", xo, o1), ("h2", Xd, h2), ("a", Xf, a2), ("x", xd, x2)):
        print("chain", tag, rel(gpu.cpu(), ref.cpu()))
    print("rms x0 %.3e  o1 %.3e  x %.3e  |a@Wd| %.3e" % (x0.pow(2).mean().sqrt(), o1.pow(2).mean().sqrt(), x2.pow(2).mean().sqrt(), (a2 @ Wd.t()).pow(2).mean().sqrt()))
