mkdir -p gpurun_out/r2n
for i in 1 2; do timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "dsv3_decode_device_mode or private_round_one_rank" > gpurun_out/r2n/pytest_$i.log 2>&1; tail -3 gpurun_out/r2n/pytest_$i.log; grep FAILED gpurun_out/r2n/pytest_$i.log; done
TXB_NO_PDL=1 timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "dsv3_decode_device_mode" > gpurun_out/r2n/pytest_nopdl.log 2>&1; tail -2 gpurun_out/r2n/pytest_nopdl.log; grep FAILED gpurun_out/r2n/pytest_nopdl.log
