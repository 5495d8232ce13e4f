# round 2 session r (4 GPUs): fused kernels signal their own completion (gs_peer_wait instead of
# two fence kernels); full GPU suite (incl. the torchrun multi-GPU test), parity, benches
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r2r_pytest_n$N.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2r_pytest_n$N.log; grep -E "^FAILED" gpurun_out/r2r_pytest_n$N.log | head
timeout 600 $R --master-port 29901 tests/mgpu_check.py > gpurun_out/r2r_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 gpurun_out/r2r_check_n$N.log | cut -c1-600
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=zero,ordered,ordered_hier timeout 600 $R --master-port 29902 tests/mgpu_check.py > gpurun_out/r2r_check_n${N}_r50.log 2>&1; echo "check r50 rc=$?"; tail -n 1 gpurun_out/r2r_check_n${N}_r50.log | cut -c1-400
B="--no-cpu-baseline --steps 20 --warmup 5 --no-allreduce-sweep --no-e2e"
for i in 1 2; do
  timeout 300 $R --master-port 2991$i bench.py --gpus $N $B > gpurun_out/r2r_bench_n${N}_zero_$i.log 2>&1; echo "zero $i rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*\|"nvlink": {[^}]*}' gpurun_out/r2r_bench_n${N}_zero_$i.log
done
timeout 300 $R --master-port 29915 bench.py --gpus $N --model alexnet $B > gpurun_out/r2r_bench_n${N}_zero_alexnet.log 2>&1; echo "alexnet rc=$?"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2r_bench_n${N}_zero_alexnet.log
