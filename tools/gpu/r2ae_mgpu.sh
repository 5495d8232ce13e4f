# round 2 session ae (4 GPUs): the driver's scaling commands on the final tree (default args, N = 1, 2, 4) + reference arm
export PYTHONPATH=.
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python bench.py > $O/r2ae_bench_n1.log 2>&1; echo "n1 rc=$?"; grep -o '"value": [0-9.]*' $O/r2ae_bench_n1.log | head -1
P=29920
for N in 2 4; do
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N > $O/r2ae_bench_n$N.log 2>&1; echo "n$N rc=$?"; grep -o '"value": [0-9.]*\|"ms_per_step": [0-9.]*' $O/r2ae_bench_n$N.log | head -2
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --impl reference --gpus $N --steps 3 --warmup 3 > $O/r2ae_ref_n$N.log 2>&1; echo "ref n$N rc=$?"; grep -o '"value": [0-9.]*' $O/r2ae_ref_n$N.log | head -1
done
