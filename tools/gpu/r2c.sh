# round 2 session c: emulation tests, all GPU tests, smoke, bench, ncu
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_emulated.py -q --timeout 900 -p no:cacheprovider > gpurun_out/r2c_emul.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_emul.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider --deselect tests/test_gpu_emulated.py > gpurun_out/r2c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench2.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv $B > gpurun_out/r2c_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lars_pass|lars_trust' -s 9 -c 3 -o gpurun_out/r2c_prof $B > gpurun_out/r2c_ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_ncu_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_ncu_smoke.log
for f in gpurun_out/r2c_emul.log gpurun_out/r2c_pytest.log gpurun_out/r2c_smoke.log gpurun_out/r2c_bench.log gpurun_out/r2c_ncu_smoke.log; do echo "== $f"; tail -n 3 $f | cut -c1-400; done
