mkdir -p gpurun_out/r2p
for i in 1 2 3 4 5 6 7 8 9 10; do timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "dsv3_decode_device_mode or private_round_one_rank or golden_one_rank" > gpurun_out/r2p/stress_$i.log 2>&1; tail -1 gpurun_out/r2p/stress_$i.log; done
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2p/pytest.log 2>&1; tail -2 gpurun_out/r2p/pytest.log
timeout 600 python bench.py > gpurun_out/r2p/bench_default.json 2> gpurun_out/r2p/bench_default.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r2p/bench_ep2.json 2> gpurun_out/r2p/bench_ep2.err
for f in gpurun_out/r2p/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'eager', d.get('p50_eager_us'), 'span', d.get('p50_kernel_span_us'), 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'), d['clocks'])"; done
tail -5 gpurun_out/r2p/bench_default.err
