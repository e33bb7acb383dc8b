#!/bin/bash
# A/B timing of library variants on the C5 probe (200k paths), alternating runs.
#   bash tools/ab.sh TAG lib1.so lib2.so ...   (paths relative to the package dir)
TAG=$1; shift
mkdir -p gpurun_out
for rep in ${AB_REPS:-1 2}; do
  for l in "$@"; do
    echo -n "$l rep$rep " >> gpurun_out/ab_${TAG}.log
    NID_LIB=paper_1804_03807_b200/$l timeout 300 python tools/probe_c5.py 200000 2>&1 | grep '"P"' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['counters']['kernel_ms_track'],2), round(d['tflops_track'],3), d['counts'])" >> gpurun_out/ab_${TAG}.log
  done
done
cat gpurun_out/ab_${TAG}.log
