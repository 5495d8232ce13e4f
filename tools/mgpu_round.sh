#!/bin/bash
# multi-GPU session: parity check + bench at N = number of visible GPUs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-mg}
PORT=29600
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $R --master-port $((PORT+1)) tests/mgpu_check.py > gpurun_out/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_check_${TAG}_n$N.log
timeout 600 $R --master-port $((PORT+2)) bench.py --gpus $N --algorithm ring > gpurun_out/bench_${TAG}_n${N}_ring.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_n${N}_ring.log
timeout 600 $R --master-port $((PORT+3)) bench.py --gpus $N --algorithm ordered --no-allreduce-sweep > gpurun_out/bench_${TAG}_n${N}_ordered.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_n${N}_ordered.log
timeout 600 $R --master-port $((PORT+4)) bench.py --gpus $N --algorithm zero --no-allreduce-sweep > gpurun_out/bench_${TAG}_n${N}_zero.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_n${N}_zero.log
