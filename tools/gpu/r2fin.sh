# round 2 final 1-GPU session on the final tree: full GPU suite, smoke, bench, reference arm, launch list
export PYTHONPATH=.
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/r2fin_pytest.log 2>&1; echo "rc=$?" >> $O/r2fin_pytest.log
tail -n 3 $O/r2fin_pytest.log; grep -E "^FAILED" $O/r2fin_pytest.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2fin_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 $O/r2fin_smoke.log
timeout 600 python bench.py > $O/r2fin_bench.log 2>&1; echo "bench rc=$?"
grep -o '"value": [0-9.]*\|"phases_ms": {[^}]*}\|"e2e": {[^}]*}\|"frac": [0-9.]*' $O/r2fin_bench.log
timeout 600 python bench.py > $O/r2fin_bench2.log 2>&1; echo "bench2 rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/r2fin_bench2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2fin_ref.log 2>&1; echo "ref rc=$?"; grep -o '"value": [0-9.]*' $O/r2fin_ref.log | head -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2fin_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2fin_ncu.log 2>&1; echo "ncu rc=$?"
