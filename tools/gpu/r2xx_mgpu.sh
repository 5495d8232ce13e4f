# round 2 session xx (4 GPUs): replicated update at p > 1 with pass 1 on its own stream
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
MGPU_ALGOS=ordered,ordered_push,ordered_hier,ordered_hier_push,ring,hierarchical,sharded timeout 900 $R --master-port 29861 tests/mgpu_check.py > $O/r2xx_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2xx_check_n$N.log | cut -c1-900
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=ordered,ordered_hier timeout 600 $R --master-port 29862 tests/mgpu_check.py > $O/r2xx_check_n${N}_r50.log 2>&1; echo "check r50 rc=$?"; tail -n 1 $O/r2xx_check_n${N}_r50.log | cut -c1-300
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29870
for A in ordered ring ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/r2xx_bench_n${N}_${A}_$P.log 2>&1; echo "$A rc=$?"; grep -o '"value": [0-9.]*' $O/r2xx_bench_n${N}_${A}_$P.log
done
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ordered --theta 1048576 $B > $O/r2xx_bench_n${N}_ordered_1m.log 2>&1; echo "ordered theta=1M rc=$?"; grep -o '"value": [0-9.]*' $O/r2xx_bench_n${N}_ordered_1m.log
