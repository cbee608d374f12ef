#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02r; mkdir -p $o
bash tools/ab.sh nl_old nle nl_u8 nl_u2 > $o/ab.txt 2>&1; cat $o/ab.txt
timeout 900 python -m pytest tests -m gpu -q -k "nonlocal or screening or damage or smoke or trajectory_c3" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
