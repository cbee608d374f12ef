#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02m; mkdir -p $o
bash tools/ab.sh base2 expl expl_xg > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c2 bash tools/ab.sh base2 expl > $o/ab_c2.txt 2>&1; cat $o/ab_c2.txt
GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/expl/libgrafem_b200.so timeout 900 python -m pytest tests -m gpu -q -k "trajectory or production_pcg or retry" > $o/pytest_expl.log 2>&1; echo "pytest expl rc=$?"; tail -3 $o/pytest_expl.log
timeout 900 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log
