# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab11
EPD_LIB_PATH=ab/bp1.so timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_encoder_gpu.py tests/test_bounds_gpu.py -x -q > gpurun_out/ab11/tests.txt 2>&1
for r in 1 2; do for v in bp0 bp1; do echo "== $v"; EPD_LIB_PATH=ab/$v.so timeout 300 python tools/small_shard.py siglip 1,2,3,10; EPD_LIB_PATH=ab/$v.so timeout 300 python tools/small_shard.py internvit 1,2,4; done; done > gpurun_out/ab11/small.txt 2>&1
