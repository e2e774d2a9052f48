#!/bin/bash
# Same-box A/B of environment settings on a short bench (engine value, e2e): bash scripts/ab_env.sh "A=1" "A=2" ...
for round in 1 2; do for v in "$@"; do
  env $v timeout 400 python bench.py --steps 256 --warmup 8 --db-batches "" --no-c1 --no-comparators --no-cpu-baseline --no-perfect > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', 'round $round', d['value'], d['e2e']['value'], d['ms_per_step'], d['steps_per_token'])" 2>&1 | tail -1
done; done
