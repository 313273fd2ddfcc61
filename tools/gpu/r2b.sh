# round 2: private-buffer round parity on 2 GPUs + first EP=1/EP=2 numbers
mkdir -p gpurun_out/r2b
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b/pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2b/bench_ep1.json 2> gpurun_out/r2b/bench_ep1.err
for P in 0 32 128; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline --private $P > gpurun_out/r2b/bench_ep2_p$P.json 2> gpurun_out/r2b/bench_ep2_p$P.err
done
tail -3 gpurun_out/r2b/pytest.log
for f in gpurun_out/r2b/bench*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d['config'].get('private_tokens'))"; done
