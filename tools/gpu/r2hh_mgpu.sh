# round 2 session hh (4 GPUs): step times with the 4M-cycle pre-step sleep
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29930
for A in zero ordered ring zero ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A $B > $O/r2hh_bench_n${N}_${A}_$P.log 2>&1; echo "$A rc=$?"; grep -o '"value": [0-9.]*' $O/r2hh_bench_n${N}_${A}_$P.log
done
