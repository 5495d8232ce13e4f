# round 2 session jj (2 GPUs): LL small-bucket kernel in the pipeline (padded bucket ranges)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_pipeline.py tests/test_gpu_overlap.py tests/test_gpu_dropin.py -q -x --timeout 600 -p no:cacheprovider > $O/r2jj_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/r2jj_pytest.log; grep -E "^FAILED" $O/r2jj_pytest.log | head -3
MGPU_ALGOS=ordered,ordered_push,ordered_hier,ordered_hier_push,ordered_inc,ordered_host,ordered_busy timeout 900 $R --master-port 29941 tests/mgpu_check.py > $O/r2jj_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2jj_check_n$N.log | cut -c1-900
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29950
for T in 262144 1048576 16777216; do
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ordered --theta $T $B > $O/r2jj_bench_n${N}_ordered_$T.log 2>&1; echo "ordered theta=$T rc=$?"; grep -o '"value": [0-9.]*\|"buckets": [0-9]*' $O/r2jj_bench_n${N}_ordered_$T.log | tr '\n' ' '; echo
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N --algorithm ring --theta $T $B > $O/r2jj_bench_n${N}_ring_$T.log 2>&1; echo "ring theta=$T rc=$?"; grep -o '"value": [0-9.]*' $O/r2jj_bench_n${N}_ring_$T.log
done
