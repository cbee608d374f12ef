#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02u; mkdir -p $o
bash tools/ab.sh cur red > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c1 bash tools/ab.sh cur red > $o/ab_c1.txt 2>&1; cat $o/ab_c1.txt
CONFIG=c2 bash tools/ab.sh cur red > $o/ab_c2.txt 2>&1; cat $o/ab_c2.txt
GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/red/libgrafem_b200.so timeout 900 python -m pytest tests -m gpu -q -k "trajectory or production_pcg or retry or solve_error or graph" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
