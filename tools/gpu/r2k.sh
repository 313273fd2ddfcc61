# 4-GPU verification: full gpu suite, bench at EP=1/2/4 for decode / kimi / prefill, stamps at EP=4,
# reference arm at EP=4, KV paced + clock probe
mkdir -p gpurun_out/r2k
nvidia-smi -L > gpurun_out/r2k/gpus.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k/pytest.log
tail -16 gpurun_out/r2k/pytest.log
timeout 300 python tools/debug/clock_probe.py > gpurun_out/r2k/clock_probe.txt 2>&1; cat gpurun_out/r2k/clock_probe.txt | tail -6
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2k/kv_paced.json 2>&1; tail -c 700 gpurun_out/r2k/kv_paced.json
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for CFG in decode kimi prefill; do
  timeout 300 python bench.py --config $CFG --steps 100 --warmup 10 > gpurun_out/r2k/bench_${CFG}_ep1.json 2> gpurun_out/r2k/bench_${CFG}_ep1.err
  for N in 2 4; do
    timeout 400 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config $CFG --gpus $N --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2k/bench_${CFG}_ep$N.json 2> gpurun_out/r2k/bench_${CFG}_ep$N.err
  done
done
timeout 300 $TR --nproc-per-node 4 --master-port 29650 tools/prof_torchrun.py --reps 50 --private 0 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/r2k/stamps_decode_ep4.txt
timeout 600 $TR --nproc-per-node 4 --master-port 29660 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/r2k/ref_ep4.json 2> gpurun_out/r2k/ref_ep4.err
for f in gpurun_out/r2k/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['kernel_us'], 'span', d.get('p50_kernel_span_us'), 'eager', d.get('p50_eager_us'), 'e2e', d['e2e']['value'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
tail -c 400 gpurun_out/r2k/ref_ep4.json
