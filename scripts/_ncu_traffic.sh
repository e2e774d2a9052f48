mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python scripts/sanitize_step.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none -k regex:sk_gemm --csv --log-file gpurun_out/gemm_traffic.csv python scripts/profile_step.py --steps 2 > gpurun_out/traffic.log 2>&1; echo "traffic rc=$?"; tail -2 gpurun_out/traffic.log
