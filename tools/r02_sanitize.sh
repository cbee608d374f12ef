#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/sanitize; mkdir -p $o
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py > $o/$tool.log 2>&1; echo "$tool rc=$?"; tail -3 $o/$tool.log
done
