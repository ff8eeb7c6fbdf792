#!/bin/bash
# A/B of the backward list chunk size (ISOGS_CHUNK) on configs 3 and 2 and the
# emulated W=8 band; parity tests first.
mkdir -p gpurun_out
python -m pytest tests/test_train_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for ck in ${CHUNKS:-0 512}; do for cfg in config3 config2; do
ISOGS_CHUNK=$ck python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 > gpurun_out/ck${ck}_$cfg.json 2> gpurun_out/ck.log
python -c "import json;d=json.load(open('gpurun_out/ck${ck}_$cfg.json'));print('chunk=$ck $cfg', round(d['value'],1), {k:round(v,3) for k,v in d['phases_ms'].items() if k.startswith('raster') or k=='tile_offsets'}, round(d['roofline']['frac'],3))" || tail -5 gpurun_out/ck.log
done
ISOGS_CHUNK=$ck python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/emul_ck$ck.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/emul_ck$ck.json'));print('chunk=$ck emulW8', [round(x,3) for x in d['per_rank_compute_ms']], round(d['projected_images_per_s'],1), {k:round(v,3) for k,v in d['per_rank_mean_phases_ms'][3].items()})"
done
