#!/bin/bash
# BASELINE configs 3 and 4 on one B200 (all stages logical on one device):
#   C3: Llama-2-13B shape, 1/2/4/8 stages (1 = GPU greedy decode), tree width w and
#       branching k sweeps at 8 stages (the tree's depth in flight = the stage count)
#   C4: Llama-2-70B shape bf16, 8 stages, 4096-token prompt, 7B-shape draft model forward
# Every SpecPipe line also runs the auto draft model (68M shape for 13B).
mkdir -p gpurun_out
out=gpurun_out/config_sweep.jsonl
: > $out
run() { timeout 900 python bench.py --db-batches "" --no-cpu-baseline --no-comparators --no-perfect --no-c1 "$@" 2>>gpurun_out/config_sweep.err | tail -1 >> $out; echo "done $*: rc=$?"; }
run --model 13b --stages 1 --steps 64
for st in 2 4 8; do run --model 13b --stages $st --w 64 --k 16 --steps 256 --warmup 8; done
for w in 16 128; do run --model 13b --stages 8 --w $w --k 16 --steps 256 --warmup 8; done
for k in 4 8 32; do run --model 13b --stages 8 --w 64 --k $k --steps 256 --warmup 8; done
run --model 70b --stages 8 --w 64 --k 16 --prompt-len 4096 --steps 96 --warmup 4 --profile-steps 8
python - <<'PY'
import json
for line in open("gpurun_out/config_sweep.jsonl"):
    line = line.strip()
    if not line.startswith("{"):
        print("bad line", line[:200]); continue
    d = json.loads(line); c = d["config"]
    if c["stages"] == 1:
        print(f"{c['model']:45s} stages=1 (greedy decode) prompt={c['prompt_len']}: TBT {d['value']:.3f} ms/token, "
              f"roofline {d['step_roofline']['frac']:.3f}")
        continue
    print(f"{c['model']:45s} stages={c['stages']} w={c['w']} k={c['k']} prompt={c['prompt_len']}: TBT {d['value']:.3f} "
          f"ms/token (e2e {d['e2e']['value']:.3f}), {d['ms_per_step']:.3f} ms/step, steps/token {d['steps_per_token']}, "
          f"step roofline {d['step_roofline']['frac']:.3f}, K2 {d['roofline']['frac']:.3f}, "
          f"draft model {(c.get('draft_model') or 'none')[:16]}")
PY
