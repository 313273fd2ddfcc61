mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests/test_moe_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2q/pytest.log 2>&1; tail -2 gpurun_out/r2q/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q/smoke.log 2>&1; tail -1 gpurun_out/r2q/smoke.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2q/bench_ep1.json 2> gpurun_out/r2q/bench_ep1.err
timeout 300 python bench.py --config kimi --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2q/bench_kimi_ep1.json 2> gpurun_out/r2q/bench_kimi_ep1.err
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2q/stamps_ep1.txt 2>&1
for f in gpurun_out/r2q/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"; done
grep -v nan gpurun_out/r2q/stamps_ep1.txt | grep "CTA" | head -24
