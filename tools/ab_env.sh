#!/bin/bash
# A/B timing of one library under environment variants on the C5 probe (200k paths).
#   bash tools/ab_env.sh TAG "VAR=1" "" ...   ("" = the default environment)
TAG=$1; shift
mkdir -p gpurun_out
for rep in ${AB_REPS:-1 2}; do
  for e in "$@"; do
    echo -n "[${e:-default}] rep$rep " >> gpurun_out/ab_${TAG}.log
    env $e timeout 300 python tools/probe_c5.py 200000 2>&1 | grep '"P"' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['counters']['kernel_ms_track'],2), round(d['tflops_track'],3), d['counts'])" >> gpurun_out/ab_${TAG}.log
  done
done
cat gpurun_out/ab_${TAG}.log
