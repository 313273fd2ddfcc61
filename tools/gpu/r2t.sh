mkdir -p gpurun_out/r2t
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/r2t/kv_vec.json 2>&1; tail -c 250 gpurun_out/r2t/kv_vec.json; echo
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 --grid 148 > gpurun_out/r2t/kv_vec_g148.json 2>&1; tail -c 250 gpurun_out/r2t/kv_vec_g148.json; echo
timeout 600 python tools/bench_kv.py --steps 20 --no-tma > gpurun_out/r2t/kv_steps_vec.json 2>&1; tail -c 300 gpurun_out/r2t/kv_steps_vec.json; echo
timeout 600 python tools/bench_weights.py > gpurun_out/r2t/weights.json 2>&1; tail -c 700 gpurun_out/r2t/weights.json; echo
timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/r2t/pytest_engine.log 2>&1; tail -2 gpurun_out/r2t/pytest_engine.log
