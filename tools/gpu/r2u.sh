mkdir -p gpurun_out/r2u
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2u/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/r2u/pytest_checked.log; tail -3 gpurun_out/r2u/pytest_checked.log
grep -c "txb check failed" gpurun_out/r2u/pytest_checked.log
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 300 python -c "
import ctypes as C, torch, sys
sys.path.insert(0,'.')
from paper_2510_27656_b200 import _lib
v=C.c_uint32(0); _lib.call('txb_check_failures', 0, C.byref(v)); print('checked build flag', hex(v.value))
" >> gpurun_out/r2u/pytest_checked.log 2>&1; tail -1 gpurun_out/r2u/pytest_checked.log
timeout 600 python tools/bench_weights.py > gpurun_out/r2u/weights.json 2>&1; tail -c 500 gpurun_out/r2u/weights.json
