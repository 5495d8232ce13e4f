# round 2 session f: pass-1 L2 bulk prefetch A/B
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_emulated.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default pf0 pf2 pf1m3 default pf0; do
  if [ $v = default ]; then L=""; else L="GRADSYNC_B200_LIB=paper_1807_11205_b200/_lib/variants/libgradsync_b200_$v.so"; fi
  env $L timeout 300 $B > gpurun_out/r2f_bench_$v.log 2>&1
  echo "== $v"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2f_bench_$v.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:lars_pass1' -s 3 -c 1 -o gpurun_out/r2f_prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak > gpurun_out/r2f_ncu.log 2>&1
tail -n 2 gpurun_out/r2f_pytest.log
