for k in 0,1 0,2 1,1 1,2 0,4; do echo "knobs $k"; python bench.py --db-batches "" --steps 32 --no-cpu-baseline --attn-knobs $k 2>/dev/null | python -c "
import sys, json
for line in sys.stdin:
    d=json.loads(line); t=d['gpu_kernel_ms_per_step']; print(' value',d['value'],'ms/step',d['ms_per_step'], {k:v for k,v in t.items() if k.startswith('attn')})"; done
