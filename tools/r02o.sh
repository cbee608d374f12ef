#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02o; mkdir -p $o
bash tools/ab.sh cur h1 h2 > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c2 bash tools/ab.sh cur h1 h2 > $o/ab_c2.txt 2>&1; cat $o/ab_c2.txt
