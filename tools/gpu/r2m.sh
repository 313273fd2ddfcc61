mkdir -p gpurun_out/r2m
timeout 300 python tools/debug/clock_probe.py > gpurun_out/r2m/clock_probe_cold.txt 2>&1; tail -5 gpurun_out/r2m/clock_probe_cold.txt
timeout 300 python tools/debug/clock_probe.py --warm > gpurun_out/r2m/clock_probe_warm.txt 2>&1; tail -5 gpurun_out/r2m/clock_probe_warm.txt
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2m/kv_paced.json 2>&1; tail -c 900 gpurun_out/r2m/kv_paced.json
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2m/pytest.log 2>&1; tail -2 gpurun_out/r2m/pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2m/bench_ep1.json 2> gpurun_out/r2m/bench_ep1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2m/bench_ep2.json 2> gpurun_out/r2m/bench_ep2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/prof_torchrun.py --reps 50 > gpurun_out/r2m/stamps_ep2.txt 2>&1
for f in gpurun_out/r2m/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'eager', d.get('p50_eager_us'), 'span', d.get('p50_kernel_span_us'), 'wflush', d.get('p50_write_flush_us'), 'b2b', d.get('p50_back_to_back_us'), d.get('back_to_back'))"; done
grep -v nan gpurun_out/r2m/stamps_ep2.txt | grep "CTA" | head -24
