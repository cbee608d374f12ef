#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02k; mkdir -p $o
CONFIG=c4 STEPS=5 bash tools/ab.sh dyn512 dyn768 dyn512g12 dyn384g12 dyn512g6 dyn512nc > $o/ab_c4.txt 2>&1; cat $o/ab_c4.txt
timeout 900 python -m pytest tests -m gpu -q -k "large_matrix or production_pcg or c4" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
