# compute-sanitizer evidence: memcheck + synccheck on the 1-GPU
# kernels and the emulated multi-rank kernels, racecheck on the shared-memory
# reductions (pass 1 / trust / pass 2 / rs_pass1).  Small shapes: the tools
# slow kernels down by 10-100x.
export PYTHONPATH=.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
T="python -m pytest -q -p no:cacheprovider --timeout 1200"
SEL1="tests/test_gpu_pipeline.py::test_odd_sizes_and_unaligned_segments tests/test_gpu_pipeline.py::test_non_power_of_two_workers_and_scale tests/test_gpu_pipeline.py::test_config1_ordered_matches_reference_golden tests/test_gpu_dropin.py"
SEL2="tests/test_gpu_emulated.py::test_sharded_fused_step_bit_exact tests/test_gpu_emulated.py::test_ordered_allreduce_step_bit_exact tests/test_gpu_emulated.py::test_hierarchical_allreduce_bit_exact tests/test_gpu_emulated.py::test_reduce_scatter_and_allgather_bit_exact tests/test_gpu_f32wire.py"
for tool in memcheck synccheck; do
  timeout 2400 $CS --tool $tool --error-exitcode 86 --print-limit 20 --target-processes all $T $SEL1 > gpurun_out/sanitize/${tool}_lars.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize/${tool}_lars.log
  timeout 2400 $CS --tool $tool --error-exitcode 86 --print-limit 20 --target-processes all $T $SEL2 > gpurun_out/sanitize/${tool}_peer.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize/${tool}_peer.log
done
timeout 2400 $CS --tool racecheck --racecheck-report all --error-exitcode 86 --print-limit 20 --target-processes all $T tests/test_gpu_pipeline.py::test_config1_ordered_matches_reference_golden "tests/test_gpu_emulated.py::test_sharded_fused_step_bit_exact[2]" > gpurun_out/sanitize/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize/racecheck.log
for f in gpurun_out/sanitize/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
