#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  SANITIZE_C4=$([ $tool = memcheck ] && echo 1) timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.txt
done
