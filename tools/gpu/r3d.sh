# after the receive-table race fix: release + checked suites on 4 GPUs, bench EP=1/2/4 decode
mkdir -p gpurun_out/r3d
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3d/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3d/pytest.log
tail -3 gpurun_out/r3d/pytest.log
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3d/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/r3d/pytest_checked.log; tail -3 gpurun_out/r3d/pytest_checked.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py > gpurun_out/r3d/bench_decode_ep1.json 2> gpurun_out/r3d/bench_decode_ep1.err
for N in 2 4; do for CFG in decode kimi; do
  timeout 600 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config $CFG --gpus $N > gpurun_out/r3d/bench_${CFG}_ep$N.json 2> gpurun_out/r3d/bench_${CFG}_ep$N.err
done; done
for f in gpurun_out/r3d/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'), 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
