#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02q; mkdir -p $o
bash tools/ab.sh cur diag > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c2 bash tools/ab.sh cur diag > $o/ab_c2.txt 2>&1; cat $o/ab_c2.txt
GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/diag/libgrafem_b200.so timeout 900 python -m pytest tests -m gpu -q -k "trajectory or production_pcg or retry or solve_error" > $o/pytest_diag.log 2>&1; echo "pytest diag rc=$?"; tail -3 $o/pytest_diag.log
