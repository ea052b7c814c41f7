# scratch GPU script for the current A/B round (overwritten per experiment)
mkdir -p gpurun_out/ab2
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_encoder_gpu.py tests/test_bounds_gpu.py -x -q > gpurun_out/ab2/tests.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --launch-skip 37 --launch-count 7 -o gpurun_out/ab2/full_c2_layer python tools/one_step.py siglip 10 > gpurun_out/ab2/ncu_full.log 2>&1
for w in c2 c5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-prefill --steps 30 2>/dev/null | tail -n 1; done > gpurun_out/ab2/bench.txt
