mkdir -p gpurun_out/r2l
timeout 300 python tools/debug/clock_probe.py > gpurun_out/r2l/clock_probe.txt 2>&1; tail -6 gpurun_out/r2l/clock_probe.txt
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2l/kv_paced.json 2>&1; tail -c 900 gpurun_out/r2l/kv_paced.json
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2l/bench_ep1.json 2> gpurun_out/r2l/bench_ep1.err
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2l/stamps_ep1.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2l/bench_ep2.json 2> gpurun_out/r2l/bench_ep2.err
timeout 900 python -m pytest tests/test_moe_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2l/pytest_moe.log 2>&1; tail -2 gpurun_out/r2l/pytest_moe.log
for f in gpurun_out/r2l/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d.get('p50_eager_us'), d.get('p50_kernel_span_us'), d.get('p50_write_flush_us'))"; done
grep -v nan gpurun_out/r2l/stamps_ep1.txt | grep "CTA" | head -24
