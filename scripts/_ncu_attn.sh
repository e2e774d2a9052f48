mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"attn_(tile|shared)" -s 1 -c 4 -o gpurun_out/attn2 -f python scripts/profile_step.py --steps 1 > gpurun_out/attn2.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/attn2.log
