#!/bin/bash
# Quick multi-GPU session: parity (incl. incremental API and push-form ordered
# all-reduce), step benches per algorithm, whole-gradient busBW, size sweep.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-mq}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 500 $R --master-port 29641 tests/mgpu_check.py > $O/mgpu_check_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n$N.log
GS_ORDERED_PUSH=1 MGPU_ALGOS=ordered,ordered_inc timeout 300 $R --master-port 29642 tests/mgpu_check.py > $O/mgpu_check_${TAG}_n${N}_push.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n${N}_push.log
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep"
P=29650
for A in zero ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/bench_${TAG}_n${N}_$A.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_$A.log
done
P=$((P+1)); GS_ORDERED_PUSH=1 timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ordered $B > $O/bench_${TAG}_n${N}_ordered_push.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_ordered_push.log
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ring --no-cpu-baseline --steps 5 --warmup 3 --no-e2e > $O/bench_${TAG}_n${N}_busbw.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_busbw.log
P=$((P+1)); timeout 600 $R --master-port $P tools/allreduce_sweep.py --variants ring,ordered,ordered_push --min-log2 16 --out $O/sweep_${TAG}_n$N.jsonl > $O/sweep_${TAG}_n$N.log 2>&1; echo "rc=$?" >> $O/sweep_${TAG}_n$N.log
if [ "${RSAB:-0}" = "1" ]; then
  P=$((P+1)); GS_RS_MODE=inbox timeout 300 $R --master-port $P bench.py --gpus $N --algorithm zero $B > $O/bench_${TAG}_n${N}_zero_inbox.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_inbox.log
  P=$((P+1)); GS_RS_MODE=inbox MGPU_ALGOS=zero timeout 300 $R --master-port $P tests/mgpu_check.py > $O/mgpu_check_${TAG}_n${N}_inbox.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n${N}_inbox.log
  P=$((P+1)); GS_RS_STAGE=1 timeout 300 $R --master-port $P bench.py --gpus $N --algorithm zero $B > $O/bench_${TAG}_n${N}_zero_stage.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_stage.log
  P=$((P+1)); GS_RS_STAGE=1 MGPU_ALGOS=zero,zero_inc timeout 300 $R --master-port $P tests/mgpu_check.py > $O/mgpu_check_${TAG}_n${N}_stage.log 2>&1; echo "rc=$?" >> $O/mgpu_check_${TAG}_n${N}_stage.log
fi
if [ "${ZTHETA:-0}" = "1" ]; then
  for T in 1048576 4194304 67108864; do
    P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm zero --theta $T $B --no-e2e > $O/bench_${TAG}_n${N}_zero_theta$T.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_theta$T.log
  done
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm zero --model alexnet $B > $O/bench_${TAG}_n${N}_zero_alexnet.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_alexnet.log
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm zero --overflow $B --no-e2e > $O/bench_${TAG}_n${N}_zero_overflow.log 2>&1; echo "rc=$?" >> $O/bench_${TAG}_n${N}_zero_overflow.log
fi
