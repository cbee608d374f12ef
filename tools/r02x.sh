#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02x; mkdir -p $o
CONFIG=c4 STEPS=5 bash tools/ab.sh ch1 ch2 ch4 > $o/ab_c4.txt 2>&1; cat $o/ab_c4.txt
GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/ch4/libgrafem_b200.so timeout 900 python -m pytest tests -m gpu -q -k "large_matrix" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $o/pytest.log
timeout 300 python tools/cg_trace_pipe.py c3 > $o/trace_c3.txt 2>&1; cat $o/trace_c3.txt
