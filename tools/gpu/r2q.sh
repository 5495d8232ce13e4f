# round 2 session q: gs_lars_fused (whole p = 1 update in one persistent kernel)
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r2q_pytest_pipe.log 2>&1; echo "pipeline pytest rc=$?"; tail -n 3 gpurun_out/r2q_pytest_pipe.log; grep -E "^FAILED|Error" gpurun_out/r2q_pytest_pipe.log | head -5
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in fused nofused fused nofused; do
  X=""; [ $v = nofused ] && X="--no-fused-step"
  timeout 300 $B $X > gpurun_out/r2q_bench_$v.log 2>&1; echo "== $v rc=$?"
  grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"gpu_launches": [0-9]*\|"frac": [0-9.]*' gpurun_out/r2q_bench_$v.log
done
timeout 300 python bench.py --model alexnet --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2q_bench_alexnet.log 2>&1; echo "== alexnet"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2q_bench_alexnet.log
timeout 300 python bench.py --overflow --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2q_bench_overflow.log 2>&1; echo "== overflow"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2q_bench_overflow.log
P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak"
timeout 600 ncu --cache-control all --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:lars_ -s 2 -c 4 --csv $P > gpurun_out/r2q_ncu_traffic.csv 2>&1
grep -E "dram__bytes|hit_rate|gpu__time" gpurun_out/r2q_ncu_traffic.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(const.*)//' | head -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lars_fused -s 2 -c 1 -o gpurun_out/r2q_prof $P > gpurun_out/r2q_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/r2q_pytest_all.log 2>&1; echo "all gpu pytest rc=$?"; tail -n 2 gpurun_out/r2q_pytest_all.log
