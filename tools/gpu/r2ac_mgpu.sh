# round 2 session ac (4 GPUs): ordered kernel grid A/B for 256 KB-8 MB buckets (MIN_ELEMS_PER_CTA)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
P=29890
for M in 16384 4096 1024 16384 4096 1024; do
  P=$((P+1)); GS_AB_SCRIPT=tools/allreduce_sweep.py GS_MIN_ELEMS_PER_CTA=$M timeout 300 $R --master-port $P tools/ab_small_cap.py --min-log2 18 --max-log2 23 --variants ordered,ordered_push > $O/r2ac_sweep_m${M}_$P.log 2>&1; echo "sweep M=$M rc=$?"
  grep '"variant"' $O/r2ac_sweep_m${M}_$P.log | python -c "import sys,json; print(' '.join('%s/%d:%.1f' % (r['variant'][8:] or 'pull', r['bytes']>>10, r['us']) for r in map(json.loads, sys.stdin)))"
done
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e --algorithm ordered"
for M in 16384 4096 16384 4096; do
for T in 262144 1048576; do
  P=$((P+1)); GS_MIN_ELEMS_PER_CTA=$M timeout 300 $R --master-port $P tools/ab_small_cap.py --gpus $N --theta $T $B > $O/r2ac_bench_m${M}_t${T}_$P.log 2>&1; echo "bench M=$M theta=$T rc=$?"; grep -o '"value": [0-9.]*' $O/r2ac_bench_m${M}_t${T}_$P.log
done
done
