# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab6
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab6/tests.txt 2>&1
for r in 1 2 3; do for v in t0 t8; do EPD_LIB_PATH=ab/$v.so timeout 120 python tools/attn_ab.py; done; done > gpurun_out/ab6/attn.txt 2>&1
for r in 1 2; do for v in t0 t8; do for w in c5; do echo "$v $w"; EPD_LIB_PATH=ab/$v.so timeout 300 python bench.py --workload $w --no-cpu-baseline --no-prefill --steps 30 2>/dev/null | tail -n 1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['achieved'],d['clocks'])"; done; done; done > gpurun_out/ab6/bench.txt 2>&1
for v in t0 t8; do EPD_LIB_PATH=ab/$v.so timeout 300 python tools/small_shard.py internvit 1,2,4,13; done > gpurun_out/ab6/small.txt 2>&1
