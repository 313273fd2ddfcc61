mkdir -p gpurun_out/r2j
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2j/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2j/pytest.log
tail -3 gpurun_out/r2j/pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2j/bench_ep1.json 2> gpurun_out/r2j/bench_ep1.err
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2j/stamps_ep1.txt 2>&1
for P in 0 32; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline --private $P > gpurun_out/r2j/bench_ep2_p$P.json 2> gpurun_out/r2j/bench_ep2_p$P.err
done
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2j/kv_paced.json 2>&1
for f in gpurun_out/r2j/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d.get('p50_eager_us'), d.get('p50_kernel_span_us'), d.get('p50_write_flush_us'), d['config'].get('private_tokens'))"; done
tail -c 800 gpurun_out/r2j/kv_paced.json
