#!/bin/bash
# compute-sanitizer memcheck / racecheck over scripts/sanitize_step.py configs (one GPU).
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > $out
for tool in memcheck racecheck; do
  for cfg in mha gqa draft; do
    small=""; [ $tool = racecheck ] && small="TP_SANITIZE_SMALL=1"
    res=$(env $small timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_step.py $cfg 2>&1 | grep -E "sanitize step ok|ERROR SUMMARY|RACECHECK SUMMARY|Error|Invalid|Hazard" | sort | uniq -c | head -8 | tr '\n' ' ')
    echo "== $tool $cfg ${small}: $res" >> $out
  done
done
cat $out
