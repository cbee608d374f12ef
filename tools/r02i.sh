#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02i; mkdir -p $o
bash tools/ab.sh base xg g2 g6 matl2 xg_g6 > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c1 bash tools/ab.sh base xg g2 g6 > $o/ab_c1.txt 2>&1; cat $o/ab_c1.txt
