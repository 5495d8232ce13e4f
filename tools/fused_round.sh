#!/bin/bash
# fused-collective session: parity (zero fused + unfused) + bench both at N GPUs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-fz}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
MGPU_ALGOS=${MGPU_ALGOS:-zero,zero_unfused,ordered} timeout 400 $R --master-port 29611 tests/mgpu_check.py > gpurun_out/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_check_${TAG}_n$N.log
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero timeout 400 $R --master-port 29612 tests/mgpu_check.py > gpurun_out/mgpu_check_${TAG}_n${N}_r50.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_check_${TAG}_n${N}_r50.log
for A in zero zero_unfused ordered; do
  timeout 300 $R --master-port 29613 bench.py --gpus $N --algorithm $A --no-allreduce-sweep --no-cpu-baseline > gpurun_out/bench_${TAG}_n${N}_$A.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_n${N}_$A.log
done
