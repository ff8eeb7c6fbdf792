set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_peer_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -15
timeout 1500 python -m pytest tests/test_dist_scale_gpu.py -x -q -k "True" 2>&1 | tail -8
for ex in peer nccl; do
for c in config2 config3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29611 bench.py --dist --exchange $ex --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/dist1_${ex}_${c}.json 2> gpurun_out/dist1_${ex}_${c}.log
tail -c 400 gpurun_out/dist1_${ex}_${c}.json; echo
done; done
