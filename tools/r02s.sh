#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02s; mkdir -p $o
bash tools/ab.sh cur ntn ntn2 > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c4 STEPS=5 bash tools/ab.sh cur ntn2 > $o/ab_c4.txt 2>&1; cat $o/ab_c4.txt
GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/ntn2/libgrafem_b200.so timeout 900 python -m pytest tests -m gpu -q -k "forces or stiffness or system or trajectory or high_valence or fused" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
