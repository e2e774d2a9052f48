#!/bin/bash
# Same-box A/B of environment settings on the emulated stage-per-GPU bench (bench.py --emulate-gpus N).
N=${N:-8}
for round in 1 2; do for v in "$@"; do
  env $v timeout 600 python bench.py --emulate-gpus $N --steps 128 --warmup 8 --db-batches "" --no-c1 --no-comparators --no-cpu-baseline --no-perfect > gpurun_out/emu.json 2> gpurun_out/emu.err
  python -c "import json;d=json.load(open('gpurun_out/emu.json'));print('$v round $round', d['value'], d['e2e']['value'], d['ms_per_step'], d['e2e_host_ms_per_step'])" 2>&1 | tail -1
done; done
