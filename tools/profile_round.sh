#!/bin/bash
# Round-end measurements into gpurun_out/r02 (copied into profiles/r02 afterwards):
# bench lines of every workload, the reference arm, the N = 2 path on one GPU, ncu launch
# lists and one-layer full captures of C2 / C5, small-shard encode times.
set -x
python -m paper_2501_05460_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/r02
timeout 600 python bench.py > gpurun_out/r02/bench_c2.log 2>&1
timeout 600 python bench.py --workload c5 > gpurun_out/r02/bench_c5.log 2>&1
timeout 600 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/r02/bench_c4.log 2>&1
timeout 600 python bench.py --workload c4w --no-cpu-baseline > gpurun_out/r02/bench_c4w.log 2>&1
timeout 600 python bench.py --workload c2i --no-cpu-baseline > gpurun_out/r02/bench_c2i.log 2>&1
timeout 600 python bench.py --workload c2s --steps 5 > gpurun_out/r02/bench_c2s.log 2>&1
timeout 600 python bench.py --workload c2p --steps 3 > gpurun_out/r02/bench_c2p.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r02/bench_ref.log 2>&1
EPD_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --no-prefill > gpurun_out/r02/bench_n2_onegpu.log 2>&1
timeout 300 python tools/small_shard.py siglip 1,2,3,5,10 > gpurun_out/r02/small_shard.txt 2>&1
timeout 300 python tools/small_shard.py internvit 1,2,4,13 >> gpurun_out/r02/small_shard.txt 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_c2.csv python tools/one_step.py siglip 10 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_c5.csv python tools/one_step.py internvit 13 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --launch-skip 37 --launch-count 7 -o gpurun_out/r02/full_c2_layer python tools/one_step.py siglip 10 > gpurun_out/r02/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off --launch-skip 33 --launch-count 7 -o gpurun_out/r02/full_c5_layer python tools/one_step.py internvit 13 > gpurun_out/r02/ncu_full5.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench/xu_rate.cu -o /tmp/xu_rate && /tmp/xu_rate > gpurun_out/r02/xu_rate.txt 2>&1
ls gpurun_out/r02
