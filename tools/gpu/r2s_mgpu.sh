# round 2 session s (4 GPUs): completion signals with one system fence per CTA vs PDL-launched fence kernels
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
MGPU_ALGOS=zero,zero_inc,zero_host timeout 600 $R --master-port 29931 tests/mgpu_check.py > gpurun_out/r2s_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 gpurun_out/r2s_check_n$N.log | cut -c1-400
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
P=29940
for v in sig fence sig fence; do
  X=""; [ $v = fence ] && X="--no-done-signals"
  P=$((P+1)); timeout 300 $R --master-port $P bench.py --gpus $N $B $X > gpurun_out/r2s_bench_n${N}_$v.log 2>&1; echo "== $v rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2s_bench_n${N}_$v.log
done
