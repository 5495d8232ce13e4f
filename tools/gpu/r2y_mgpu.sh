# round 2 session y (4 GPUs): one-shot small-bucket all-reduce
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_pipeline.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r2y_pytest.log; grep -E "^FAILED" gpurun_out/r2y_pytest.log | head -3
MGPU_ALGOS=ordered,ordered_push,ordered_inc,ordered_host,ordered_busy timeout 600 $R --master-port 29991 tests/mgpu_check.py > gpurun_out/r2y_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 gpurun_out/r2y_check_n$N.log | cut -c1-600
timeout 900 $R --master-port 29992 tools/allreduce_sweep.py --min-log2 10 --max-log2 26 --out gpurun_out/r2y_sweep_n$N.jsonl > gpurun_out/r2y_sweep_n$N.log 2>&1; echo "sweep rc=$?"; grep summary gpurun_out/r2y_sweep_n$N.log
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/r2y_sweep_n4.jsonl') if '"variant"' in l]
by={}
for r in rows: by.setdefault(r['bytes'],{})[r['variant']]=round(r['us'],1)
for b in sorted(by): print(b, by[b])
PY
