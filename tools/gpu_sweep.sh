#!/bin/bash
# Workload sweep on one B200 (bench lines without the CPU leg) and the
# emulated multi-GPU per-rank timings.  Outputs under gpurun_out/sweep/.
mkdir -p gpurun_out/sweep
B="--steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0"
python bench.py --config config2 $B > gpurun_out/sweep/config2.json 2>> gpurun_out/sweep/log
python bench.py --config config4 $B > gpurun_out/sweep/config4.json 2>> gpurun_out/sweep/log
python bench.py --config config3 --res 1024 $B > gpurun_out/sweep/config3res1024.json 2>> gpurun_out/sweep/log
python bench.py --config config3 --res 4096 $B > gpurun_out/sweep/config3res4096.json 2>> gpurun_out/sweep/log
for w in 2 4 8; do python tools/emulated_ranks.py --config config3 --workers $w > gpurun_out/sweep/emul3_w$w.json 2>> gpurun_out/sweep/log; done
python tools/emulated_ranks.py --config config2 --workers 8 > gpurun_out/sweep/emul2_w8.json 2>> gpurun_out/sweep/log
for w in 4 8; do python tools/emulated_ranks.py --config config4 --workers $w > gpurun_out/sweep/emul4_w$w.json 2>> gpurun_out/sweep/log; done
for r in 1024 4096; do python tools/emulated_ranks.py --config config3 --res $r --workers 8 > gpurun_out/sweep/emul3_res${r}_w8.json 2>> gpurun_out/sweep/log; done
ls -la gpurun_out/sweep
