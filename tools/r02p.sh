#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02p; mkdir -p $o
bash tools/ab.sh cur co_pcg co_dmg > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c4 STEPS=5 bash tools/ab.sh cur co_pcg > $o/ab_c4.txt 2>&1; cat $o/ab_c4.txt
