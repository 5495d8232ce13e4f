# round 2 session o: persisting-L2 set-aside + evict_last (h4, h5), grad-norm-off pass-1 A/B
export PYTHONPATH=.
mkdir -p gpurun_out
V=paper_1807_11205_b200/_lib/variants
for v in h4 h5; do
  GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2o_pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -n 1 gpurun_out/r2o_pytest_$v.log
done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default nognorm h4 h5 default nognorm h4 h5; do
  X=""; L=""
  if [ $v = nognorm ]; then X="--no-grad-norm"; elif [ $v != default ]; then L="GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so"; fi
  env $L timeout 300 $B $X > gpurun_out/r2o_bench_$v.log 2>&1
  echo "== $v"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2o_bench_$v.log; grep "set-aside" gpurun_out/r2o_bench_$v.log | head -1
done
for v in h4 h5; do
  for cc in none all; do
  GRADSYNC_B200_LIB=$V/libgradsync_b200_$v.so timeout 600 ncu --cache-control $cc --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:lars_pass -s 6 -c 4 --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak > gpurun_out/r2o_ncu_${v}_$cc.csv 2>&1
  echo "== ncu $v cache-control $cc"; grep -E "dram__bytes|hit_rate|gpu__time" gpurun_out/r2o_ncu_${v}_$cc.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(const.*)//' | head -8
  done
done
