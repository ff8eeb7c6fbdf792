rm -rf gpurun_out/ab; mkdir -p gpurun_out/ab
VAR=ISOGS_CHUNK VALS="0 1048576 2048 1024 512" bash tools/ab_env.sh
for v in 1024 512; do ISOGS_CHUNK=$v timeout 600 python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/ab/emul_ck$v.json 2>>gpurun_out/ab/log; python -c "import json;d=json.load(open('gpurun_out/ab/emul_ck$v.json'));print('emul ck$v', round(d['projected_images_per_s'],1), round(d['step_compute_max_ms'],3), [round(r['backward_fold'],3) for r in d['per_rank_mean_phases_ms']])"; done
