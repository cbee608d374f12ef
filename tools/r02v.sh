#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02v; mkdir -p $o
bash tools/ab.sh cur red > $o/ab.txt 2>&1; cat $o/ab.txt
