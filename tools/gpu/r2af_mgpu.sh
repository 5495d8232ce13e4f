# round 2 session af (4 GPUs): full GPU suite on the final tree (incl. the torchrun test) + every mgpu_check algorithm
export PYTHONPATH=.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/r2af_pytest.log 2>&1; echo "rc=$?" >> $O/r2af_pytest.log
tail -n 3 $O/r2af_pytest.log; grep -E "^FAILED" $O/r2af_pytest.log | head
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29931 tests/mgpu_check.py > $O/r2af_check_n$N.log 2>&1; echo "check rc=$?"; tail -n 1 $O/r2af_check_n$N.log | cut -c1-1500
