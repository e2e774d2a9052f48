"""Diagnostics: where does the GPU Llama path depart from the oracle at the 7B shape?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2504_04104_b200 as tp
from paper_2504_04104_b200.model import KvCache, LlamaConfig, LlamaModel, prefill_rows
from oracle.llama import LlamaOracle


def rel(a, b):
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.abs(d).max() / np.abs(b).max()), float(np.sqrt((d * d).mean() / (np.asarray(b, np.float64) ** 2).mean()))


def f32(u16):
    return (np.asarray(u16).astype(np.uint32) << 16).view(np.float32)


name = sys.argv[1] if len(sys.argv) > 1 else "7b"
cfg = {"7b": LlamaConfig.llama2_7b(), "13b": LlamaConfig.llama2_13b(), "70b": LlamaConfig.llama2_70b()}[name]
m = LlamaModel(cfg, max_nodes=64, layer_range=(0, 1), with_embed=True, with_head=False)
o = LlamaOracle(cfg.vocab, cfg.hidden, cfg.layers, cfg.heads, cfg.kv_heads, cfg.ffn, layer_range=(0, 1), with_head=False)
rng = np.random.default_rng(0)
for P in (8, 64, 512):
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, P)]
    c = KvCache(cfg.layers, cfg.hidden, capacity=P + 8).bind(m, (0, 1))
    xg = prefill_rows(m, c, prompt, layer_range=(0, 1)).cpu().numpy()
    kv = o.new_dense_kv(P + 8)
    xo = o.prefill_block(prompt, kv)
    kg, vg = f32(c.keys[0]), f32(c.values[0])
    print(P, "K", rel(kg, kv.keys(0)), "V", rel(vg, kv.values(0)), "x", rel(xg, xo),
          "x first8", rel(xg[:8], xo[:8]), "x last8", rel(xg[-8:], xo[-8:]))
    # per-row worst
    d = np.abs(xg - xo).max(axis=1) / np.abs(xo).max()
    print("   worst rows", np.argsort(d)[-5:], np.sort(d)[-5:])
    # exact K equality fraction
    print("   K bitwise-equal frac", float((kg == kv.keys(0)).mean()), "V", float((vg == kv.values(0)).mean()))
