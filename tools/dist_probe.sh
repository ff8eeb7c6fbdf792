#!/bin/bash
# Sharded-engine timing probes on one GPU (world 1): plain env launch vs torchrun.
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_PORT=29514 OMP_NUM_THREADS=1 \
  python bench.py --gpus 1 --steps 5 --warmup 3 --dist --no-cpu-baseline > gpurun_out/probe_env_omp1.json 2> gpurun_out/probe_env_omp1.log
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_PORT=29516 \
  python bench.py --gpus 1 --steps 5 --warmup 3 --dist --no-cpu-baseline > gpurun_out/probe_env.json 2> gpurun_out/probe_env.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29515 \
  bench.py --gpus 1 --steps 5 --warmup 3 --dist --no-cpu-baseline > gpurun_out/probe_trun.json 2> gpurun_out/probe_trun.log
for f in probe_env_omp1 probe_env probe_trun; do echo "== $f"; grep -E '^\{' gpurun_out/$f.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],2), d['phases_ms'])"; done
