mkdir -p gpurun_out/r2i
timeout 300 python tools/debug/clock_probe.py > gpurun_out/r2i/clock_probe.txt 2>&1
cat gpurun_out/r2i/clock_probe.txt | tail -8
timeout 300 python bench.py --steps 100 --warmup 10 > gpurun_out/r2i/bench_ep1.json 2> gpurun_out/r2i/bench_ep1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i/launches_ep1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2i/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dispatch_roles|k_combine_fused" -s 40 -c 2 -o gpurun_out/r2i/ep1_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2i/ncu_full.log 2>&1
tail -3 gpurun_out/r2i/ncu_full.log
python -c "import json; d=json.loads(open('gpurun_out/r2i/bench_ep1.json').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d.get('p50_eager_us'), d.get('p50_kernel_span_us'), d['roofline'], d['e2e']['value'], d.get('cpu_baseline',{}).get('value'))"
