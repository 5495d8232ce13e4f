#!/bin/bash
# End-of-round multi-GPU session: parity for every algorithm, the default
# bench line, every algorithm's step, AlexNet, theta sweep, skip path,
# whole-gradient busBW, the message-size sweep, and NCCL pinned to Ring / NVLS.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-fin}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
P=29900
timeout 500 $R --master-port $((P+1)) tests/mgpu_check.py > $O/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n$N.log
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero,ordered timeout 400 $R --master-port $((P+2)) tests/mgpu_check.py > $O/mgpu_check_${TAG}_n${N}_r50.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n${N}_r50.log
P=$((P+3)); timeout 300 $R --master-port $P bench.py --gpus $N > $O/bench_${TAG}_n${N}_default.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_default.log
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep"
for A in zero_unfused ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/bench_${TAG}_n${N}_$A.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_$A.log
done
if [ $N -ge 4 ]; then
  for A in hierarchical sharded; do
    P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A --group-size 2 $B > $O/bench_${TAG}_n${N}_${A}_k2.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_${A}_k2.log
  done
fi
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet $B > $O/bench_${TAG}_n${N}_zero_alexnet.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_alexnet.log
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet --algorithm ring $B > $O/bench_${TAG}_n${N}_ring_alexnet.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_ring_alexnet.log
for T in 262144 4194304 67108864; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --theta $T $B --no-e2e > $O/bench_${TAG}_n${N}_zero_theta$T.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_theta$T.log
done
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --overflow $B --no-e2e > $O/bench_${TAG}_n${N}_zero_overflow.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_overflow.log
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ring --no-cpu-baseline --steps 5 --warmup 3 --no-e2e > $O/bench_${TAG}_n${N}_busbw.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_busbw.log
P=$((P+1)); timeout 900 $R --master-port $P tools/allreduce_sweep.py --out $O/sweep_${TAG}_n$N.jsonl > $O/sweep_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n$N.log
P=$((P+1)); NCCL_ALGO=Ring timeout 600 $R --master-port $P tools/allreduce_sweep.py --variants ring --min-log2 20 --out $O/sweep_${TAG}_n${N}_ncclring.jsonl > $O/sweep_${TAG}_n${N}_ncclring.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n${N}_ncclring.log
P=$((P+1)); NCCL_ALGO=NVLS timeout 600 $R --master-port $P tools/allreduce_sweep.py --variants ring --min-log2 20 --out $O/sweep_${TAG}_n${N}_ncclnvls.jsonl > $O/sweep_${TAG}_n${N}_ncclnvls.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n${N}_ncclnvls.log
