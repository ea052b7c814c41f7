# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab8
EPD_LIB_PATH=ab/s1.so timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/ab8/tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/ab8/tests.txt
if grep -q "passed" gpurun_out/ab8/tests.txt && ! grep -q "failed" gpurun_out/ab8/tests.txt; then
for r in 1 2 3; do for v in s0 s1; do EPD_LIB_PATH=ab/$v.so timeout 120 python tools/attn_ab.py; done; done > gpurun_out/ab8/attn.txt 2>&1
fi
