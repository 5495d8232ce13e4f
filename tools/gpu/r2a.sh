set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a_base.log 2>&1
GS_P2_REVERSE=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a_rev.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a_base2.log 2>&1
GS_P2_REVERSE=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a_rev2.log 2>&1
GS_P2_REVERSE=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --model alexnet > gpurun_out/r2a_rev_alex.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --model alexnet > gpurun_out/r2a_base_alex.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1
tail -3 gpurun_out/r2a_pytest.log
