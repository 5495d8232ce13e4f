# round 2 session zz (4 GPUs): LL cap 256 KB -> 512 KB (θ = 256 KiB buckets take the LL kernel)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q > $O/r2zz_pytest_emulated.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/r2zz_pytest_emulated.log
MGPU_THETA=262144 MGPU_ALGOS=ordered,ordered_push,ordered_hier,ordered_hier_push,ring,sharded timeout 900 $R --master-port 29861 tests/mgpu_check.py > $O/r2zz_check_n${N}_256k.log 2>&1; echo "check 256k rc=$?"; tail -n 1 $O/r2zz_check_n${N}_256k.log | cut -c1-900
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29870
for T in 262144 1048576; do
for A in ordered ring ordered ring; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm $A --theta $T $B > $O/r2zz_bench_n${N}_${A}_${T}_$P.log 2>&1; echo "$A theta=$T rc=$?"; grep -o '"value": [0-9.]*' $O/r2zz_bench_n${N}_${A}_${T}_$P.log
done
done
