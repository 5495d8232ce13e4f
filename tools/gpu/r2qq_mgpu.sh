# round 2 session qq: gs_zero_update bench (after the bench phase-name fix)
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
echo skip-pytest
echo skip-check
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
for i in 1 2 3; do
  timeout 300 $R --master-port 2992$((i+3)) bench.py --gpus $N $B > gpurun_out/r2qq_bench_n${N}_$i.log 2>&1; echo "zero $i rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*' gpurun_out/r2qq_bench_n${N}_$i.log
done
