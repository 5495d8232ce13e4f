#!/bin/bash
# zero (sharded fused step) robustness: parity + benches at theta 16 MiB and 64 MiB, both RS forms
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-zc}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep"
P=29800
MGPU_ALGOS=zero,zero_inc,ordered timeout 300 $R --master-port $((P+1)) tests/mgpu_check.py > $O/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n$N.log
MGPU_MODEL=resnet50 MGPU_THETA=67108864 MGPU_ALGOS=zero timeout 300 $R --master-port $((P+2)) tests/mgpu_check.py > $O/mgpu_check_${TAG}_n${N}_r50_64m.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n${N}_r50_64m.log
P=$((P+1)); GS_MULTICAST=0 timeout 300 $R --master-port $P bench.py --gpus $N $B > $O/bench_${TAG}_n${N}_zero_nomc.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_nomc.log
for T in ${THETAS:-16777216 67108864}; do
  for M in ${MODES:-pull inbox}; do
    P=$((P+3)); GS_RS_MODE=$M timeout 300 $R --master-port $P bench.py --gpus $N --theta $T $B > $O/bench_${TAG}_n${N}_zero_${M}_theta$T.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_${M}_theta$T.log
  done
done
