# round 2 multi-GPU session: real-NVLink parity of every algorithm after the
# rank-table ABI refactor, benches, whole-gradient busBW, message sweep
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r2g}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
P=29700
timeout 600 $R --master-port $((P+1)) tests/mgpu_check.py > $O/${TAG}_check_n$N.log 2>&1; echo "rc=$?" >> $O/${TAG}_check_n$N.log
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero,ordered,ordered_hier timeout 600 $R --master-port $((P+2)) tests/mgpu_check.py > $O/${TAG}_check_n${N}_r50.log 2>&1; echo "rc=$?" >> $O/${TAG}_check_n${N}_r50.log
P=$((P+3)); timeout 400 $R --master-port $P bench.py --gpus $N > $O/${TAG}_bench_n${N}_zero.log 2>&1; echo "rc=$?" >> $O/${TAG}_bench_n${N}_zero.log
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep"
for A in zero_unfused ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/${TAG}_bench_n${N}_$A.log 2>&1; echo "rc=$?" >> $O/${TAG}_bench_n${N}_$A.log
done
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet $B > $O/${TAG}_bench_n${N}_zero_alexnet.log 2>&1; echo "rc=$?" >> $O/${TAG}_bench_n${N}_zero_alexnet.log
P=$((P+1)); timeout 900 $R --master-port $P tools/allreduce_sweep.py --min-log2 14 --out $O/${TAG}_sweep_n$N.jsonl > $O/${TAG}_sweep_n$N.log 2>&1; echo "rc=$?" >> $O/${TAG}_sweep_n$N.log
for f in $O/${TAG}_check_n$N.log $O/${TAG}_check_n${N}_r50.log; do echo "== $f"; tail -n 2 $f | cut -c1-2500; done
for f in $O/${TAG}_bench_n${N}_*.log; do echo "== $f"; grep -o '"value": [0-9.]*' $f | head -1; grep -o '"phases_ms": {[^}]*}' $f; done
grep summary $O/${TAG}_sweep_n$N.log
