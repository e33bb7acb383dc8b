#!/bin/bash
# Evidence run for profiles/: reference arm, torchrun launch, ncu launch list, one full-set capture.
set -x
mkdir -p gpurun_out
python bench.py --impl reference --steps 2 --warmup 1 --ref-sample 96 > gpurun_out/ref_arm.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/torchrun1.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python tools/probe_c5.py 200000 > gpurun_out/plain_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:track_ctl -c 1 -o gpurun_out/prof_track_r01 \
  python tools/probe_c5.py 200000 > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ref_arm.log gpurun_out/torchrun1.log gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
