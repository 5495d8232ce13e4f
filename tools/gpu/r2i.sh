# round 2 session i: executor, full GPU suite, bench, overlap timeline, sanitizers
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
tail -n 3 gpurun_out/r2i_pytest.log; grep -E "^FAILED" gpurun_out/r2i_pytest.log | head
timeout 600 python bench.py > gpurun_out/r2i_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_bench.log
grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"e2e": {[^}]*}' gpurun_out/r2i_bench.log
timeout 600 python tools/overlap_timeline.py --out gpurun_out/r2i_overlap > gpurun_out/r2i_overlap.json 2> gpurun_out/r2i_overlap.err; echo "rc=$?"; cat gpurun_out/r2i_overlap.json | head -40
timeout 3000 bash tools/gpu/sanitize.sh
