mkdir -p gpurun_out/r2y
timeout 900 python -m pytest tests/test_moe_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2y/pytest.log 2>&1; tail -2 gpurun_out/r2y/pytest.log
timeout 300 python tools/prof_torchrun.py --reps 50 --noflush 2>&1 | grep -v nan | grep CTA | head -26
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2y/bench_ep1.json 2> gpurun_out/r2y/bench_ep1.err
python -c "import json,sys; d=json.loads(open('gpurun_out/r2y/bench_ep1.json').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'), d['roofline'].get('kernel_span_us'), d['roofline'].get('frac_on_span'))"
