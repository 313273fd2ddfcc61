mkdir -p gpurun_out/kv3
timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/kv3/ready.json 2>&1
timeout 300 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/kv3/paced.json 2>&1
timeout 300 python tools/bench_kv_stream.py --modes ready --reps 2 --tma > gpurun_out/kv3/ready_tma.json 2>&1
for m in ready paced ready_tma; do python -c "
import json; d=json.loads(open('gpurun_out/kv3/$m.json').read().strip().splitlines()[-1]); print('$m', d['best_ms'], d['best_gbs'], d['frac_of_peak'], d['all_bytes_identical'], [r.get('last_tick_to_end_us') for r in d['runs']])"; done
