for opt in "--no-perfect" "" ; do timeout 900 python bench.py --no-cpu-baseline $opt 2>/dev/null | python -c "
import sys, json
for line in sys.stdin:
    d=json.loads(line); print('opt=$opt value',d['value'], [ (r['batch'], r['tokens_per_s'], r['ms_per_tick']) for r in d['specpipe_db']['results']])"; done
timeout 600 python scripts/bench_db.py --batches 1,16,1 | cut -c1-120
