# round 2 session rr (4 GPUs): gs_zero_update at p = 4
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
MGPU_ALGOS=zero,zero_inc,zero_host,zero_busy timeout 600 $R --master-port 29881 tests/mgpu_check.py > $O/r2rr_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2rr_check_n$N.log | cut -c1-500
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero timeout 600 $R --master-port 29882 tests/mgpu_check.py > $O/r2rr_check_n${N}_r50.log 2>&1; echo "check r50 rc=$?"; tail -n 1 $O/r2rr_check_n${N}_r50.log | cut -c1-300
P=29883
for i in 1 2 3; do
  P=$((P+1)); timeout 400 $R --master-port $P bench.py --gpus $N > $O/r2rr_bench_n${N}_zero_$i.log 2>&1; echo "zero $i rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*\|"nvlink": {[^}]*}' $O/r2rr_bench_n${N}_zero_$i.log
done
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --model alexnet $B > $O/r2rr_bench_n${N}_zero_alexnet.log 2>&1; echo "alexnet rc=$?"; grep -o '"value": [0-9.]*' $O/r2rr_bench_n${N}_zero_alexnet.log
