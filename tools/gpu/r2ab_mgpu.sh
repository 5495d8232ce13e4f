# round 2 session ab (4 GPUs): LL cap A/B at θ = 256 KiB (old 128 K elements vs new 256 K)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e --algorithm ordered --theta 262144"
P=29880
for C in 131072 262144 131072 262144; do
  P=$((P+1)); GS_LL_MAX_ELEMS=$C GS_SMALL_CAP_ELEMS=$C timeout 300 $R --master-port $P tools/ab_small_cap.py --gpus $N $B > $O/r2ab_n${N}_cap${C}_$P.log 2>&1; echo "cap=$C rc=$?"; grep -o '"value": [0-9.]*' $O/r2ab_n${N}_cap${C}_$P.log
done
