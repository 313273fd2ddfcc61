# KV stream booking batch A/B: 32 (shipped) vs 128 vs 1024 steps per fence
mkdir -p gpurun_out/kvb
for L in libtxb200.so libtxb200_b128.so libtxb200_b1024.so; do
  TXB200_LIB=$PWD/paper_2510_27656_b200/$L timeout 300 python tools/bench_kv_stream.py --modes ready --reps 3 > gpurun_out/kvb/ready_$L.json 2>&1
  TXB200_LIB=$PWD/paper_2510_27656_b200/$L timeout 300 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/kvb/paced_$L.json 2>&1
  python -c "
import json
for m in ('ready','paced'):
    d=json.loads(open(f'gpurun_out/kvb/{m}_$L.json').read().strip().splitlines()[-1]); print('$L', m, d['best_ms'], d['best_gbs'], d['all_bytes_identical'], [r.get('last_tick_to_end_us') for r in d['runs']])"
done
