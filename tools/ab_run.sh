# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab3
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_encoder_gpu.py tests/test_bounds_gpu.py -x -q > gpurun_out/ab3/tests.txt 2>&1
for r in 1 2; do for v in prev new_nobulk new; do EPD_LIB_PATH=ab/$v.so timeout 120 python tools/ln_ab.py; EPD_LIB_PATH=ab/$v.so timeout 120 python tools/gemm_ab.py; done; done > gpurun_out/ab3/micro.txt 2>&1
for r in 1 2; do for v in prev new; do for w in c2 c5; do echo "$v $w"; EPD_LIB_PATH=ab/$v.so timeout 300 python bench.py --workload $w --no-cpu-baseline --no-prefill --steps 30 2>/dev/null | tail -n 1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['achieved'],d['clocks'])"; done; done; done > gpurun_out/ab3/bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --launch-skip 37 --launch-count 7 -o gpurun_out/ab3/full_c2_layer python tools/one_step.py siglip 10 > gpurun_out/ab3/ncu_full.log 2>&1
