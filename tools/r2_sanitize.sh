#!/bin/bash
O=${OUT:-gpurun_out/r2san}; mkdir -p $O
python tools/sanitize_case.py > $O/plain.log 2>&1; echo rc=$? >> $O/plain.log
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --target-processes all python tools/sanitize_case.py > $O/$tool.log 2>&1
  echo rc=$? >> $O/$tool.log
done
