# round 2 session p (4 GPUs): NVLink peer-access probe; zero / ordered benches with the device-sleep timing
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $R --master-port 29811 tools/nvlink_probe.py > gpurun_out/r2p_probe_n$N.log 2>&1; echo "probe rc=$?"
grep '^{' gpurun_out/r2p_probe_n$N.log | tail -n 60
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
for A in zero ordered; do
  timeout 300 $R --master-port 2982$((RANDOM % 9)) bench.py --gpus $N --algorithm $A $B > gpurun_out/r2p_bench_n${N}_$A.log 2>&1; echo "$A rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*' gpurun_out/r2p_bench_n${N}_$A.log
done
