mkdir -p gpurun_out/w
timeout 300 python tools/debug/weights_prepare_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex.sum --clock-control none -c 6 python tools/debug/weights_prepare_probe.py 2>&1 | grep -E "k_amax|k_quant|gpu__time|dram__|lts__" | tail -10
timeout 300 python tools/bench_weights.py > gpurun_out/w/weights2.json 2>&1; tail -c 800 gpurun_out/w/weights2.json
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "weight or prepare or quant" 2>&1 | tail -2
