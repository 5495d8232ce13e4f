# round 2 session w (4 GPUs): push form of the own two-level (hierarchical) all-reduce
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_emulated.py -q -x --timeout 300 -p no:cacheprovider -k hierarchical > gpurun_out/r2w_pytest.log 2>&1; echo "emulated hier pytest rc=$?"; tail -n 1 gpurun_out/r2w_pytest.log
MGPU_ALGOS=ordered_hier,ordered_hier_push,ordered_push timeout 600 $R --master-port 29961 tests/mgpu_check.py > gpurun_out/r2w_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 gpurun_out/r2w_check_n$N.log | cut -c1-500
MGPU_MODEL=resnet50 MGPU_THETA=16777216 MGPU_ALGOS=ordered_hier_push timeout 600 $R --master-port 29962 tests/mgpu_check.py > gpurun_out/r2w_check_n${N}_r50.log 2>&1; echo "check r50 rc=$?"; tail -n 1 gpurun_out/r2w_check_n${N}_r50.log | cut -c1-300
for i in 1 2; do
timeout 400 $R --master-port 2997$i bench.py --gpus $N --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/r2w_bench_n${N}_$i.log 2>&1; echo "bench rc=$?"
grep '"value"' gpurun_out/r2w_bench_n${N}_$i.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['allreduce']))"
done
timeout 900 $R --master-port 29975 tools/allreduce_sweep.py --min-log2 14 --out gpurun_out/r2w_sweep_n$N.jsonl > gpurun_out/r2w_sweep_n$N.log 2>&1; echo "sweep rc=$?"; grep summary gpurun_out/r2w_sweep_n$N.log
