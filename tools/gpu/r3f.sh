# final bench lines with the final bench.py: EP=1/2/4 (decode / kimi / prefill), stamps, reference arm EP=1
mkdir -p gpurun_out/r3f
nvidia-smi -L > gpurun_out/r3f/gpus.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py > gpurun_out/r3f/bench_decode_ep1.json 2> gpurun_out/r3f/bench_decode_ep1.err
for CFG in kimi prefill; do timeout 600 python bench.py --config $CFG --no-cpu-baseline > gpurun_out/r3f/bench_${CFG}_ep1.json 2> gpurun_out/r3f/bench_${CFG}_ep1.err; done
for N in 2 4; do for CFG in decode kimi prefill; do
  timeout 600 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config $CFG --gpus $N > gpurun_out/r3f/bench_${CFG}_ep$N.json 2> gpurun_out/r3f/bench_${CFG}_ep$N.err
done; done
timeout 300 python tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/r3f/stamps_decode_ep1.txt
for N in 2 4; do timeout 300 $TR --nproc-per-node $N --master-port $((29650+N)) tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/r3f/stamps_decode_ep$N.txt; done
for f in gpurun_out/r3f/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'), 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], 'cpu', d.get('cpu_baseline',{}).get('value'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
timeout 600 python bench.py --impl reference > gpurun_out/r3f/ref_ep1.json 2> gpurun_out/r3f/ref_ep1.err; tail -c 200 gpurun_out/r3f/ref_ep1.json
