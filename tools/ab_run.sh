# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab10
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "linear_acc" > gpurun_out/ab10/tests.txt 2>&1
timeout 120 python tools/split_ab.py >> gpurun_out/ab10/tests.txt 2>&1
for r in 1 2 3; do for sp in 0 8; do echo "split $sp"; EPD_PREFILL_MAX_SPLIT=$sp timeout 300 python tools/measure_prefill_latency.py gpurun_out/ab10/pl_$sp.json 2>&1 | grep -E " 662 | 3350 "; done; done > gpurun_out/ab10/prefill.txt 2>&1
