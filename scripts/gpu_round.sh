#!/bin/bash
# One gpurun call: GPU tests, bench, optional extras.  Usage: bash scripts/gpu_round.sh [tests|bench|ncu|gemm]...
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for what in "$@"; do
  case $what in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
    tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/tests.log ;;
    bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    gemm) timeout 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; cat gpurun_out/gemm_bench.log ;;
    db) timeout 900 python scripts/bench_db.py > gpurun_out/db.log 2>&1; cat gpurun_out/db.log | tail -8 ;;
    hostprof) timeout 600 python scripts/host_profile.py > gpurun_out/hostprof.log 2>&1; head -60 gpurun_out/hostprof.log ;;
    sweep) timeout 600 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.log 2>&1; cat gpurun_out/gemm_sweep.log ;;
    launches) timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 4 > gpurun_out/prof.log 2>&1; echo "ncu rc=$?"; python scripts/launch_summary.py gpurun_out/launches.csv 4 | tee gpurun_out/launch_summary.txt ;;
    full) timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sk_gemm -s 5 -c 3 -o gpurun_out/gemm_full -f python scripts/profile_step.py --steps 2 > gpurun_out/full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/full.log ;;
  esac
done
