mkdir -p gpurun_out/r2o
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2o/pytest.log 2>&1; tail -2 gpurun_out/r2o/pytest.log
for i in 1 2 3 4 5; do timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "dsv3_decode_device_mode or private_round_one_rank" > gpurun_out/r2o/stress_$i.log 2>&1; tail -1 gpurun_out/r2o/stress_$i.log; done
/usr/bin/time -v python bench.py > gpurun_out/r2o/bench_default.json 2> gpurun_out/r2o/bench_default.err; grep -E "Elapsed" gpurun_out/r2o/bench_default.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r2o/bench_ep2.json 2> gpurun_out/r2o/bench_ep2.err
timeout 400 python bench.py --impl reference > gpurun_out/r2o/ref_ep1.json 2> gpurun_out/r2o/ref_ep1.err
for f in gpurun_out/r2o/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'eager', d.get('p50_eager_us'), 'span', d.get('p50_kernel_span_us'), 'b2b', d.get('back_to_back'), 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'), d['clocks'])"; done
tail -c 300 gpurun_out/r2o/ref_ep1.json
