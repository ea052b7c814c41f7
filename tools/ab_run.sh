# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab12
EPD_LIB_PATH=ab/db1.so timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_encoder_gpu.py tests/test_bounds_gpu.py tests/test_prefill_gpu.py -x -q > gpurun_out/ab12/tests.txt 2>&1
for r in 1 2; do for v in db0 db1; do EPD_LIB_PATH=ab/$v.so timeout 120 python tools/gemm_ab.py; done; done > gpurun_out/ab12/gemm.txt 2>&1
for r in 1 2; do for v in db0 db1; do for w in c2 c5; do echo "$v $w"; EPD_LIB_PATH=ab/$v.so timeout 300 python bench.py --workload $w --no-cpu-baseline --no-prefill --steps 30 2>/dev/null | tail -n 1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['clocks']['sm_mhz'])"; done; done; done > gpurun_out/ab12/bench.txt 2>&1
