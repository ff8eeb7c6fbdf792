# A/B of variant libraries (paper_2509_05216_b200/_build/<name>/libisogs.so; "base" = the
# default build): bench phases at configs 3 and 2.  Usage: bash tools/ab_lib.sh base name ...
mkdir -p gpurun_out/ab
for v in "$@"; do
  lib=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so
  [ $v = base ] && lib=$PWD/paper_2509_05216_b200/_build/libisogs.so
  for cfg in ${CFGS:-config3 config2}; do
    ISOGS_LIB=$lib python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 > gpurun_out/ab/lib_${v}_$cfg.json 2>>gpurun_out/ab/log
    python -c "import json;d=json.load(open('gpurun_out/ab/lib_${v}_$cfg.json'));print('$v $cfg', round(d['value'],1), {k:round(x,3) for k,x in d['phases_ms'].items() if k in ${KEYS:-('bin_emit','sort_tiles','bin_count','raster_fwd','raster_bwd')}})"
  done
done
