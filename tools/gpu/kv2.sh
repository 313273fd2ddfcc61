mkdir -p gpurun_out/kv2
timeout 120 ./tools/micro/peer_width > gpurun_out/kv2/peer_width_grid.txt 2>&1; cat gpurun_out/kv2/peer_width_grid.txt | tail -4
timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/kv2/pytest_engine.log 2>&1; tail -2 gpurun_out/kv2/pytest_engine.log
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/kv2/kv_ready.json 2>&1; tail -c 400 gpurun_out/kv2/kv_ready.json; echo
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 3 --grid 296 > gpurun_out/kv2/kv_ready_g296.json 2>&1; tail -c 300 gpurun_out/kv2/kv_ready_g296.json; echo
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/kv2/kv_paced.json 2>&1; tail -c 300 gpurun_out/kv2/kv_paced.json; echo
timeout 600 python tools/bench_kv.py --no-tma > gpurun_out/kv2/kv_step_vec.json 2>&1; tail -c 300 gpurun_out/kv2/kv_step_vec.json; echo
