# round 2 session j: overlap timeline (side stream fixed), chunk 4096 A/B
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_overlap.py -q -p no:cacheprovider > gpurun_out/r2j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest.log; tail -n 2 gpurun_out/r2j_pytest.log
timeout 600 python tools/overlap_timeline.py --out gpurun_out/r2j_overlap > gpurun_out/r2j_overlap.json 2> gpurun_out/r2j_overlap.err; echo "rc=$?"; head -30 gpurun_out/r2j_overlap.json
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in default c4096 default c4096; do
  if [ $v = default ]; then L=""; else L="GRADSYNC_B200_LIB=paper_1807_11205_b200/_lib/variants/libgradsync_b200_r2m6.so GS_CHUNK_ELEMS=4096"; fi
  env $L timeout 300 $B > gpurun_out/r2j_bench_$v.log 2>&1
  echo "== $v"; grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/r2j_bench_$v.log
done
GRADSYNC_B200_LIB=paper_1807_11205_b200/_lib/variants/libgradsync_b200_r2m6.so GS_CHUNK_ELEMS=4096 timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -p no:cacheprovider -k "resnet50_single or odd_sizes or config1" > gpurun_out/r2j_c4096_pytest.log 2>&1; tail -n 2 gpurun_out/r2j_c4096_pytest.log
