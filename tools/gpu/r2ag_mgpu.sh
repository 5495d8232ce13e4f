# round 2 session ag (2 GPUs): ordered vs NCCL ring at θ = 16 MiB / 1 MiB / 256 KiB on the final tree
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29940
for T in 16777216 1048576 262144; do
for A in ordered ring ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A --theta $T $B > $O/r2ag_bench_n${N}_${A}_${T}_$P.log 2>&1; echo "$A theta=$T rc=$?"; grep -o '"value": [0-9.]*' $O/r2ag_bench_n${N}_${A}_${T}_$P.log
done
done
