# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab4
for r in 1 2; do for v in cur sm2k sm3k; do echo "== $v"; EPD_LIB_PATH=ab/$v.so timeout 300 python tools/small_shard.py siglip 1,2,3; EPD_LIB_PATH=ab/$v.so timeout 300 python tools/small_shard.py internvit 1,2,4; done; done > gpurun_out/ab4/small.txt 2>&1
EPD_LIB_PATH=ab/sm3k.so timeout 600 python -m pytest tests/test_encoder_gpu.py -x -q > gpurun_out/ab4/tests_sm3k.txt 2>&1
