# round 2 session ii (4 GPUs): LL small-bucket all-reduce with batched polling
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_emulated.py -q -x --timeout 300 -p no:cacheprovider -k "ordered_allreduce or hier" > gpurun_out/r2ii_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r2ii_pytest.log; grep -E "^FAILED" gpurun_out/r2ii_pytest.log | head -3
timeout 900 $R --master-port 29993 tools/allreduce_sweep.py --min-log2 10 --max-log2 22 --variants ring,ordered,ordered_push,ordered_oneshot,ordered_ll --out gpurun_out/r2ii_sweep_n$N.jsonl > gpurun_out/r2ii_sweep_n$N.log 2>&1; echo "sweep rc=$?"; grep summary gpurun_out/r2ii_sweep_n$N.log; tail -3 gpurun_out/r2ii_sweep_n$N.log | cut -c1-300
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/r2ii_sweep_n4.jsonl') if '"variant"' in l]
by={}
for r in rows: by.setdefault(r['bytes'],{})[r['variant']]=(round(r['us'],1), r.get('overflow_propagated'))
for b in sorted(by): print(b, by[b])
PY
