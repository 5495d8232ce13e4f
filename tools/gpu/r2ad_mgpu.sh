# round 2 session ad (4 GPUs): push form for <= 2 MB buckets on the pull wire at p >= 4
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q > $O/r2ad_pytest_emulated.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/r2ad_pytest_emulated.log
MGPU_THETA=262144 MGPU_ALGOS=ordered,ordered_hier,ordered_busy,ordered_host timeout 900 $R --master-port 29861 tests/mgpu_check.py > $O/r2ad_check_n${N}_256k.log 2>&1; echo "check 256k rc=$?"; tail -n 1 $O/r2ad_check_n${N}_256k.log | cut -c1-900
MGPU_ALGOS=ordered,ordered_push,ordered_hier,zero,ring timeout 900 $R --master-port 29862 tests/mgpu_check.py > $O/r2ad_check_n${N}.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2ad_check_n${N}.log | cut -c1-900
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e --algorithm ordered"
P=29900
for M in 0 2097152 0 2097152; do
for T in 262144 1048576 16777216; do
  P=$((P+1)); GS_PUSH_MAX_BYTES=$M timeout 300 $R --master-port $P tools/ab_small_cap.py --gpus $N --theta $T $B > $O/r2ad_bench_m${M}_t${T}_$P.log 2>&1; echo "bench push_max=$M theta=$T rc=$?"; grep -o '"value": [0-9.]*' $O/r2ad_bench_m${M}_t${T}_$P.log
done
done
