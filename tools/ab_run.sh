# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab7
EPD_LIB_PATH=ab/ob1.so timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/ab7/tests.txt 2>&1
for r in 1 2 3; do for v in ob0 ob1; do EPD_LIB_PATH=ab/$v.so timeout 120 python tools/attn_ab.py; done; done > gpurun_out/ab7/attn.txt 2>&1
for r in 1 2; do for v in ob0 ob1; do for w in c2 c5; do echo "$v $w"; EPD_LIB_PATH=ab/$v.so timeout 300 python bench.py --workload $w --no-cpu-baseline --no-prefill --steps 30 2>/dev/null | tail -n 1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['clocks']['sm_mhz'])"; done; done; done > gpurun_out/ab7/bench.txt 2>&1
