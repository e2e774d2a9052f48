"""Tiny-model layer-0 intermediates (tp_debug_dump) vs the float32 oracle's, on a
7-token prefill: where does the GPU / oracle difference start?"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_04104_b200 as tp  # noqa: E402
from oracle.llama import LlamaOracle, bf16  # noqa: E402
from paper_2504_04104_b200 import _lib  # noqa: E402

shape = dict(vocab=512, hidden=256, layers=4, heads=2, kv_heads=1, ffn=512)
lm = tp.LlamaModel(tp.LlamaConfig(**shape), max_nodes=64)
prompt = [7, 3, 9, 1, 4, 4, 2]
n = len(prompt)
orc = LlamaOracle(**shape)
d, q, f = 256, 256, 512
dump = torch.zeros(64 * (d * 2 + q * 2 * 2 + d * 4 + d * 2 + f * 2 + d * 4), dtype=torch.uint8, device="cuda")
_lib.check(_lib.lib().tp_debug_dump(dump.data_ptr()))
cache = tp.KvCache(4, 256)
rows = tp.model.prefill_rows(lm, cache, prompt)
torch.cuda.synchronize()
o = 0


def take(nbytes, dt, shp):
    global o
    t = dump[o:o + nbytes].view(dt).reshape(shp)
    o += nbytes
    return t.float().cpu().numpy()


Xd = take(n * d * 2, torch.bfloat16, (n, d))
Xq = take(n * q * 2, torch.bfloat16, (n, q))
Xo = take(n * q * 2, torch.bfloat16, (n, q))
xo = take(n * d * 4, torch.float32, (n, d))
Xd2 = take(n * d * 2, torch.bfloat16, (n, d))
Xf = take(n * f * 2, torch.bfloat16, (n, f))
xd = take(n * d * 4, torch.float32, (n, d))
# oracle layer 0 for the same rows
w = orc.blocks[0]
x = orc.embedding[np.asarray(prompt)].astype(np.float32)
h, r = orc.norm_split_rows(x)
pos = np.arange(n)
qo = bf16(orc.rope_rows((h @ w["wq"]) * r, pos))


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-30, np.abs(b).max()))


print("Xd vs bf16(x)", rel(Xd, h))
print("Xq vs oracle", rel(Xq, qo), "frac exact", float((Xq == qo).mean()))
kv = orc.new_dense_kv(64)
for p in pos:
    kv.open_row(-1, int(p), True)
xl = orc.causal_block(0, x.copy(), kv, pos)
print("x after layer 0 vs oracle", rel(xd, xl))
h2, r2 = orc.norm_split_rows(xo)
gg = (h2 @ w["wg"]) * r2
uu = (h2 @ w["wu"]) * r2
af = bf16((gg / (1 + np.exp(-gg))) * uu)
print("Xd2 vs bf16(xo)", rel(Xd2, h2), "Xf vs oracle(from GPU xo)", rel(Xf, af), "frac exact", float((Xf == af).mean()))
print("xd vs xo + Xf@Wd", rel(xd, xo + Xf @ w["wd"]))
print("final rows vs oracle", rel(rows.float().cpu().numpy(), orc.prefill_block(prompt, orc.new_dense_kv(64))))
