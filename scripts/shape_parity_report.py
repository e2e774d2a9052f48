"""Format the JSON lines tests/test_gpu_llama_shapes.py appends to its log into
profiles/r02_llama_shape_parity.txt.

    python scripts/shape_parity_report.py gpurun_out/llama_shape_parity.jsonl > profiles/r02_llama_shape_parity.txt
"""
import json
import sys

print("# Llama parity at the benchmarked shapes (tests/test_gpu_llama_shapes.py, B200, round 2, folded RMSNorm)")
print("# e2e: GPU vs float32 oracle, (max |d| / max |oracle|, rms d / rms oracle)")
print("# per_kernel: float64 recomputation from each kernel's own GPU inputs (fraction within 1 bf16 ulp; the folded")
print("#   norm's bf16 operand within 0.5 ulp of x), or rel error; controls: distance to deliberately wrong semantics")
for line in open(sys.argv[1]):
    d = json.loads(line)
    print()
    print(f"== {d['shape']}  layers {d['layers']}  prompt {d['prompt']}")
    for k, (mx, rms) in d["e2e_errors_max_rms"].items():
        print(f"  e2e {k:22s} max {mx:.2e}  rms {rms:.2e}")
    for k, v in d["per_kernel"].items():
        print(f"  kernel {k:36s} {v:g}")
    for k, (mx, rms) in d["controls_max_rms"].items():
        print(f"  control {k:18s} max {mx:.2e}  rms {rms:.2e}")
    print(f"  argmax checked (top-1 margin > 2 TOL): {d['argmax_checked']} of 8")
