mkdir -p gpurun_out/r2g
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2g/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g/pytest.log
tail -3 gpurun_out/r2g/pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2g/bench_ep1.json 2> gpurun_out/r2g/bench_ep1.err
for P in 0 32; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline --private $P > gpurun_out/r2g/bench_ep2_p$P.json 2> gpurun_out/r2g/bench_ep2_p$P.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/prof_torchrun.py --reps 50 --private 0 > gpurun_out/r2g/stamps_ep2_p0.txt 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/r2g/kv_vec.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready,paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2g/kv_g32.json 2>&1
for f in gpurun_out/r2g/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d.get('p50_eager_us'), d.get('p50_kernel_span_us'), d.get('p50_write_flush_us'), d['config'].get('private_tokens'))"; done
