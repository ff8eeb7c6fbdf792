mkdir -p gpurun_out
python -m pytest tests/test_train_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for hf in 0 1; do for cfg in config3 config2; do
ISOGS_HEAVY_FIRST=$hf python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 > gpurun_out/hf${hf}_$cfg.json 2> gpurun_out/hf.log
python -c "import json;d=json.load(open('gpurun_out/hf${hf}_$cfg.json'));print('hf=$hf $cfg', round(d['value'],1), {k:round(v,3) for k,v in d['phases_ms'].items() if k.startswith('raster')}, round(d['roofline']['frac'],3))"
done
ISOGS_HEAVY_FIRST=$hf python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/emul_hf$hf.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/emul_hf$hf.json'));print('hf=$hf emulW8', [round(x,3) for x in d['per_rank_compute_ms']], round(d['projected_images_per_s'],1), {k:round(v,3) for k,v in d['per_rank_mean_phases_ms'][3].items()})"
done
