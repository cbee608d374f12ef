#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02g; mkdir -p $o
bash tools/ab.sh idx_eng idx_noeng r02head > $o/ab.txt 2>&1; cat $o/ab.txt
bash tools/r02_sanitize.sh
