# final 4-GPU run: release + checked suites, smoke, bench EP=1/2/4 (decode / kimi / prefill), stamps
mkdir -p gpurun_out/fin
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest.log 2>&1; echo "release rc=$? $(tail -1 gpurun_out/fin/pytest.log)"
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest_checked.log 2>&1; echo "checked rc=$? $(tail -1 gpurun_out/fin/pytest_checked.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/fin/smoke.log)"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py > gpurun_out/fin/bench_decode_ep1.json 2> gpurun_out/fin/bench_decode_ep1.err
for CFG in kimi prefill; do timeout 600 python bench.py --config $CFG --no-cpu-baseline > gpurun_out/fin/bench_${CFG}_ep1.json 2> gpurun_out/fin/bench_${CFG}_ep1.err; done
for N in 2 4; do for CFG in decode kimi prefill; do
  timeout 600 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config $CFG --gpus $N > gpurun_out/fin/bench_${CFG}_ep$N.json 2> gpurun_out/fin/bench_${CFG}_ep$N.err
done; done
timeout 300 python tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/fin/stamps_decode_ep1.txt
for N in 2 4; do timeout 300 $TR --nproc-per-node $N --master-port $((29650+N)) tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/fin/stamps_decode_ep$N.txt; done
for f in gpurun_out/fin/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'), 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
