# round 2 session b: the rank-batched peer ABI, emulation tests, smoke, bench
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_emulated.py -x -q --timeout 600 -p no:cacheprovider > gpurun_out/r2b_emul.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_emul.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider --deselect tests/test_gpu_emulated.py > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_bench.log
tail -3 gpurun_out/r2b_emul.log gpurun_out/r2b_pytest.log gpurun_out/r2b_smoke.log gpurun_out/r2b_bench.log
