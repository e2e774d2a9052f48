#!/bin/bash
# ncu evidence for profiles/: K2 DRAM traffic (launch list), full captures of K2 and the K1 kernels.
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none -k regex:sk_gemm --csv --log-file gpurun_out/gemm_traffic.csv python scripts/profile_step.py --steps 2 > gpurun_out/traffic.log 2>&1; echo "traffic rc=$?"
python scripts/gemm_traffic.py gpurun_out/gemm_traffic.csv gpurun_out/traffic.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sk_gemm -s 5 -c 3 -o gpurun_out/gemm_full -f python scripts/profile_step.py --steps 2 > gpurun_out/full.log 2>&1; echo "gemm full rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_ -s 4 -c 4 -o gpurun_out/attn_full -f python scripts/profile_step.py --steps 2 > gpurun_out/attn_full.log 2>&1; echo "attn full rc=$?"
