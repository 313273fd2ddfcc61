mkdir -p gpurun_out/r2h
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2h/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h/pytest.log
tail -25 gpurun_out/r2h/pytest.log
for P in 0 32; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline --private $P > gpurun_out/r2h/bench_ep2_p$P.json 2> gpurun_out/r2h/bench_ep2_p$P.err
done
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/r2h/kv_vec.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 --grid 296 > gpurun_out/r2h/kv_vec_g296.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 --tma > gpurun_out/r2h/kv_tma.json 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2h/kv_paced_conn32.json 2>&1
for f in gpurun_out/r2h/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d.get('p50_eager_us'), d.get('p50_kernel_span_us'), d.get('p50_write_flush_us'), d['config'].get('private_tokens'))"; done
for f in gpurun_out/r2h/kv*.json; do echo $f; tail -c 600 $f; echo; done
