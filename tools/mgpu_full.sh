#!/bin/bash
# Full multi-GPU session at N = visible GPUs: parity for every algorithm,
# ResNet-50 benches per algorithm (+ hierarchy variants), AlexNet, a theta
# sweep for the default algorithm, the forced-overflow step, and the fp16
# all-reduce message-size sweep (BASELINE config 5).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-mf}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 500 $R --master-port 29621 tests/mgpu_check.py > $O/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n$N.log
B="--no-cpu-baseline --steps 20 --warmup 5"
P=29630
for A in zero ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B --no-allreduce-sweep > $O/bench_${TAG}_n${N}_$A.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_$A.log
done
for K in 2 4; do
  if [ $K -lt $N ] && [ $((N % K)) -eq 0 ]; then
    for A in hierarchical sharded; do
      P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A --group-size $K $B --no-allreduce-sweep > $O/bench_${TAG}_n${N}_${A}_k$K.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_${A}_k$K.log
    done
  fi
done
# whole-gradient busBW of every variant (bench's own measurement, ring arm)
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ring $B > $O/bench_${TAG}_n${N}_busbw.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_busbw.log
# AlexNet (config 4)
for A in zero ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet --algorithm $A $B --no-allreduce-sweep > $O/bench_${TAG}_n${N}_alexnet_$A.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_alexnet_$A.log
done
# theta sweep (config 3), default algorithm
for T in 262144 1048576 4194304 67108864; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --theta $T $B --no-allreduce-sweep --no-e2e > $O/bench_${TAG}_n${N}_theta$T.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_theta$T.log
done
# forced overflow: the skip path
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --overflow $B --no-allreduce-sweep --no-e2e > $O/bench_${TAG}_n${N}_overflow.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_overflow.log
# message-size sweep with forced overflow (config 5)
P=$((P+1)); timeout 900 $R --master-port $P tools/allreduce_sweep.py --out $O/sweep_${TAG}_n$N.jsonl > $O/sweep_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n$N.log
P=$((P+1)); NCCL_ALGO=Ring timeout 600 $R --master-port $P tools/allreduce_sweep.py --variants ring --min-log2 20 --out $O/sweep_${TAG}_n${N}_ncclring.jsonl > $O/sweep_${TAG}_n${N}_ncclring.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n${N}_ncclring.log
P=$((P+1)); NCCL_ALGO=NVLS timeout 600 $R --master-port $P tools/allreduce_sweep.py --variants ring --min-log2 20 --out $O/sweep_${TAG}_n${N}_ncclnvls.jsonl > $O/sweep_${TAG}_n${N}_ncclnvls.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n${N}_ncclnvls.log
