mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sk_gemm -s 17 -c 5 -o gpurun_out/gemm_full -f python scripts/profile_step.py --steps 1 > gpurun_out/full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/full.log
timeout 600 ncu --set full --clock-control none -k regex:sk_gemm -s 1 -c 1 -o gpurun_out/gemm_gu48 -f python scripts/gemm_bench.py --shapes gu --n 48 --iters 1 > gpurun_out/full2.log 2>&1; echo "full2 rc=$?"; tail -2 gpurun_out/full2.log
timeout 600 ncu --set full --clock-control none -k regex:attn_tail -s 4 -c 2 -o gpurun_out/attn_full -f python scripts/profile_step.py --steps 1 > gpurun_out/full3.log 2>&1; echo "full3 rc=$?"
