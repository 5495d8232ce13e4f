#!/bin/bash
# one GPU session: tests, smoke, bench, ncu launch list + full capture of the hot kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONPATH=.
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
if [ "${NCU:-1}" = "1" ]; then
  B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-soak"
  timeout 300 $B > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $B > gpurun_out/ncu_list.log 2>&1 ; \
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lars_pass|batched_copy' -s 8 -c 6 -o gpurun_out/prof_${TAG} $B > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
if [ "${EXTRA:-0}" = "1" ]; then
  # configs 2/4 variants at N = 1: AlexNet, theta sweep, forced-overflow skip path
  B="--no-cpu-baseline --steps 20 --warmup 5"
  timeout 300 python bench.py --model alexnet $B > gpurun_out/bench_${TAG}_alexnet.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_alexnet.log
  for T in 0 262144 1048576 4194304 67108864; do
    timeout 300 python bench.py --theta $T $B --no-e2e > gpurun_out/bench_${TAG}_theta$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_theta$T.log
  done
  timeout 300 python bench.py --overflow $B --no-e2e > gpurun_out/bench_${TAG}_overflow.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_overflow.log
  timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_refarm.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_refarm.log
fi
