#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02t; mkdir -p $o
for cl in 1 0; do GF_CG_CLUSTER=$cl timeout 300 python tools/cg_trace_pipe.py c1 >> $o/trace.jsonl 2>> $o/trace.err; done
timeout 300 python tools/cg_trace_pipe.py c2 >> $o/trace.jsonl 2>> $o/trace.err
timeout 300 python tools/cg_trace_pipe.py c3 >> $o/trace.jsonl 2>> $o/trace.err
cat $o/trace.jsonl
