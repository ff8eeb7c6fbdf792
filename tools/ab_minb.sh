# backward launch bound x chunk size A/B (variant builds under _build/<name>)
mkdir -p gpurun_out/ab
for v in base mb14 mb16; do
  lib=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so
  [ $v = base ] && lib=$PWD/paper_2509_05216_b200/_build/libisogs.so
  for ck in 0 1024; do for cfg in config3 config2; do
    ISOGS_LIB=$lib ISOGS_CHUNK=$ck python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 > gpurun_out/ab/mb_${v}_${ck}_$cfg.json 2>>gpurun_out/ab/log
    python -c "import json;d=json.load(open('gpurun_out/ab/mb_${v}_${ck}_$cfg.json'));print('$v ck$ck $cfg', round(d['value'],1), {k:round(x,3) for k,x in d['phases_ms'].items() if k.startswith('raster')})"
  done; done
done
for v in mb14 mb16; do
  ISOGS_LIB=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so ISOGS_CHUNK=1024 timeout 600 python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/ab/emul_${v}.json 2>>gpurun_out/ab/log
  python -c "import json;d=json.load(open('gpurun_out/ab/emul_${v}.json'));print('emul $v ck1024', round(d['projected_images_per_s'],1), [round(r['backward_fold'],3) for r in d['per_rank_mean_phases_ms']])"
done
