mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"attn_shared" -s 2 -c 2 -o gpurun_out/attn_shared -f python scripts/profile_step.py --steps 1 > gpurun_out/attn_tail.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/attn_tail.log
