# round 2 session u: warp-specialised TMA pass 1 (2-3 consumer groups) vs the register form
export PYTHONPATH=.
mkdir -p gpurun_out
V=paper_1807_11205_b200/_lib/variants
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dropin.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2u_pytest.log; grep -E "^FAILED" gpurun_out/r2u_pytest.log | head -5
for v in g3s2 g2s3; do
  GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2u_pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -n 1 gpurun_out/r2u_pytest_$v.log
done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default notma g3s2 g2s3 default notma g3s2 g2s3; do
  L=""; [ $v != default ] && L="GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so"
  env $L timeout 300 $B > gpurun_out/r2u_bench_$v.log 2>&1; echo "== $v rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2u_bench_$v.log
done
P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lars_pass1 -s 2 -c 1 -o gpurun_out/r2u_prof $P > gpurun_out/r2u_ncu.log 2>&1; echo "ncu rc=$?"
