#!/bin/bash
# Evidence run for profiles/: default bench line, reference arm, torchrun
# launch, ncu launch list, executed FP64 instruction mix and one full-set
# capture of the tracker kernel.
#   bash tools/gpu_evidence.sh TAG
TAG=${1:-r02}
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
python bench.py --impl reference --steps 2 --warmup 1 --ref-sample 96 > gpurun_out/ref_arm_${TAG}.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-workloads > gpurun_out/torchrun_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-other-workloads > gpurun_out/ncu_launches_${TAG}.log 2>&1
python tools/probe_c5.py 200000 > gpurun_out/plain_probe_${TAG}.log 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum,gpu__time_duration.sum \
  --clock-control none -k regex:track_ -c 1 --csv --log-file gpurun_out/opmix_${TAG}.csv \
  python tools/probe_c5.py 200000 > gpurun_out/opmix_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:track_ -c 1 -o gpurun_out/prof_track_${TAG} \
  python tools/probe_c5.py 200000 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -n 2 gpurun_out/bench_${TAG}.log gpurun_out/ref_arm_${TAG}.log gpurun_out/torchrun_${TAG}.log \
  gpurun_out/ncu_launches_${TAG}.log gpurun_out/ncu_full_${TAG}.log
tail -n 8 gpurun_out/opmix_${TAG}.csv
