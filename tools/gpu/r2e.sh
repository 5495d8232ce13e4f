# round 2 session e: pass-1 variants, fp32 wire, all tests
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default c1m3 c2m2 pers3 default c2m2; do
  if [ $v = default ]; then L=""; else L="GRADSYNC_B200_LIB=paper_1807_11205_b200/_lib/variants/libgradsync_b200_$v.so"; fi
  env $L timeout 300 $B > gpurun_out/r2e_bench_$v.log 2>&1
  echo "== $v"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2e_bench_$v.log
done
tail -n 3 gpurun_out/r2e_pytest.log; grep -E "^FAILED|Error" gpurun_out/r2e_pytest.log | head
