#!/bin/bash
# Round-2 (final) evidence in one gpurun call: default bench, launch list, ncu full of K1 / K2, FlashInfer comparator.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02f_launches.csv python scripts/profile_step.py --steps 4 > gpurun_out/r02f_prof.log 2>&1; echo "launches rc=$?"
python scripts/launch_summary.py gpurun_out/r02f_launches.csv 4 > gpurun_out/r02f_launch_summary.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_ -s 4 -c 2 -o gpurun_out/r02f_attn_full -f python scripts/profile_step.py --steps 2 > gpurun_out/r02f_attn_full.log 2>&1; echo "attn full rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:sk_gemm_kernel<\\(int\\)8>" -s 8 -c 4 -o gpurun_out/r02f_gemm_full -f python scripts/profile_step.py --steps 2 > gpurun_out/r02f_gemm_full.log 2>&1; echo "gemm full rc=$?"
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none -k regex:sk_gemm --csv --log-file gpurun_out/r02f_gemm_traffic.csv python scripts/profile_step.py --steps 2 --draft-model none > gpurun_out/r02f_traffic.log 2>&1; echo "traffic rc=$?"
timeout 600 python scripts/attn_vs_flashinfer.py > gpurun_out/r02f_afi.jsonl 2>&1; timeout 600 python scripts/attn_vs_flashinfer.py --prefix 2048 >> gpurun_out/r02f_afi.jsonl 2>&1; echo "afi rc=$?"
cuobjdump -sass paper_2504_04104_b200/libtreepipe_b200.so | grep -oE "UTCHMMA|UTCBAR|UBLKCP|UTMALDG|LDTM|STTM|HMMA" | sort | uniq -c > gpurun_out/r02f_sass_ops.txt
