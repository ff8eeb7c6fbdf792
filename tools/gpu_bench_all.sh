#!/bin/bash
# Bench arms on one GPU: default N=1 line, the sharded engine at world 1
# (torchrun), and a short reference arm.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.log
echo "ours rc=$?"; tail -3 gpurun_out/bench.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --dist --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dist1.json 2> gpurun_out/dist1.log
echo "dist rc=$?"; grep -v "NCCL INFO" gpurun_out/dist1.log | tail -3; grep -c "NCCL INFO" gpurun_out/dist1.log
[ "$NO_REF" = "1" ] || { python bench.py --impl reference --steps 3 --warmup 3 --cpu-budget-s 20 > gpurun_out/ref.json 2> gpurun_out/ref.log;
echo "ref rc=$?"; tail -3 gpurun_out/ref.log; }
