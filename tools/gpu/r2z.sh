mkdir -p gpurun_out/r2z
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2z/pytest.log 2>&1; tail -2 gpurun_out/r2z/pytest.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r2z/bench_ep2.json 2> gpurun_out/r2z/bench_ep2.err
python -c "import json,sys; d=json.loads(open('gpurun_out/r2z/bench_ep2.json').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/prof_torchrun.py --reps 50 2>&1 | grep -v nan | grep CTA | head -30
