"""The draft model's top-k kernel (tp_topk_rows) vs torch.topk on 64 x 32000 fp32
logits, back-to-back launches timed with CUDA events (host-issue bound at this size:
read the kernel time from ncu: `ncu --metrics gpu__time_duration.sum -k regex:topk`)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2504_04104_b200 as tp  # noqa: E402
m = tp.LlamaModel(tp.LlamaConfig(vocab=512, hidden=256, layers=1, heads=2, kv_heads=1, ffn=512), max_nodes=16)
x = torch.randn(64, 32000, device="cuda")
for f, name in ((lambda: torch.topk(x, 16, dim=1), "torch"), (lambda: m.topk_many(x, 16), "ours")):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): f()
    e1.record(); torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1) * 10, 1), "us", flush=True)
