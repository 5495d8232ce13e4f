# round 2 session n: L2 eviction-priority A/B for pass 1 -> pass 2 (ResNet-50, 1 GPU)
export PYTHONPATH=.
mkdir -p gpurun_out
V=paper_1807_11205_b200/_lib/variants
for v in h1 h2 h3; do
  GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2n_pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -n 1 gpurun_out/r2n_pytest_$v.log
done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default h1 h2 h3 default h1 h2 h3; do
  if [ $v = default ]; then L=""; else L="GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so"; fi
  env $L timeout 300 $B > gpurun_out/r2n_bench_$v.log 2>&1
  echo "== $v"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*' gpurun_out/r2n_bench_$v.log
done
for v in default h1; do
  if [ $v = default ]; then L=""; else L="GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so"; fi
  env $L timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:lars_pass -s 6 -c 6 --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak > gpurun_out/r2n_ncu_$v.csv 2>&1
  grep -E "dram__bytes|hit_rate|gpu__time" gpurun_out/r2n_ncu_$v.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
done
