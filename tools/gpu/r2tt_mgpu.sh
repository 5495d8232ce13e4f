# round 2 session tt (4 GPUs): final multi-GPU validation of the final round-2 tree
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $O/r2tt_pytest_n$N.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/r2tt_pytest_n$N.log; grep -E "^FAILED" $O/r2tt_pytest_n$N.log | head -3
timeout 900 $R --master-port 29901 tests/mgpu_check.py > $O/r2tt_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2tt_check_n$N.log | cut -c1-2500
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero,ordered,ordered_hier,ordered_hier_push timeout 600 $R --master-port 29902 tests/mgpu_check.py > $O/r2tt_check_n${N}_r50.log 2>&1; echo "check r50 rc=$?"; tail -n 1 $O/r2tt_check_n${N}_r50.log | cut -c1-500
P=29910
for i in 1 2; do
  P=$((P+1)); timeout 400 $R --master-port $P bench.py --gpus $N > $O/r2tt_bench_n${N}_zero_$i.log 2>&1; echo "zero $i rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*\|"e2e": {[^}]*}' $O/r2tt_bench_n${N}_zero_$i.log
done
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
for A in ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/r2tt_bench_n${N}_$A.log 2>&1; echo "$A rc=$?"; grep -o '"value": [0-9.]*' $O/r2tt_bench_n${N}_$A.log
done
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet $B > $O/r2tt_bench_n${N}_zero_alexnet.log 2>&1; echo "alexnet rc=$?"; grep -o '"value": [0-9.]*' $O/r2tt_bench_n${N}_zero_alexnet.log
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --overflow $B > $O/r2tt_bench_n${N}_zero_overflow.log 2>&1; echo "overflow rc=$?"; grep -o '"value": [0-9.]*' $O/r2tt_bench_n${N}_zero_overflow.log
P=$((P+1)); timeout 1200 $R --master-port $P tools/allreduce_sweep.py --min-log2 10 --out $O/r2tt_sweep_n$N.jsonl > $O/r2tt_sweep_n$N.log 2>&1; echo "sweep rc=$?"; grep summary $O/r2tt_sweep_n$N.log
