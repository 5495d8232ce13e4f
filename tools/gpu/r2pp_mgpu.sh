# round 2 session pp: fence + trust + pass 2 push in one launch (gs_zero_update)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_checkpoint.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2pp_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r2pp_pytest.log; grep -E "^FAILED" gpurun_out/r2pp_pytest.log | head -3
MGPU_ALGOS=zero,zero_unfused,zero_inc,zero_host,zero_busy timeout 600 $R --master-port 29921 tests/mgpu_check.py > gpurun_out/r2pp_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 gpurun_out/r2pp_check_n$N.log | cut -c1-500
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
for i in 1 2 3; do
  timeout 300 $R --master-port 2992$((i+3)) bench.py --gpus $N $B > gpurun_out/r2pp_bench_n${N}_$i.log 2>&1; echo "zero $i rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*' gpurun_out/r2pp_bench_n${N}_$i.log
done
