# round 2 session k: the full GPU suite on the GS_CHECKS=1 build (device-side
# bounds / invariant asserts; compute-sanitizer is closed on this pool),
# overlap timeline on a GPU-bound backward
export PYTHONPATH=.
mkdir -p gpurun_out
GRADSYNC_B200_LIB=paper_1807_11205_b200/_lib/variants/libgradsync_b200_checks.so timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2k_checks_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_checks_pytest.log
tail -n 3 gpurun_out/r2k_checks_pytest.log; grep -E "^FAILED|gs check failed" gpurun_out/r2k_checks_pytest.log | head
timeout 900 python tools/overlap_timeline.py --out gpurun_out/r2k_overlap > gpurun_out/r2k_overlap.json 2> gpurun_out/r2k_overlap.err; echo "rc=$?"; head -40 gpurun_out/r2k_overlap.json
