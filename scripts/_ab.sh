for v in s1 s4 s1 s4; do cp paper_2504_04104_b200/lib_$v.so paper_2504_04104_b200/libtreepipe_b200.so; python bench.py --db-batches "" --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
for line in sys.stdin:
    d=json.loads(line); print('$v value',d['value'],'e2e',d['e2e']['value'], {k:v for k,v in d['gpu_kernel_ms_per_step'].items() if 'attn' in k})"; done
