#!/bin/bash
# A/B of an environment knob on the config-3 and config-2 benches:
#   VAR=ISOGS_HEAVY_PCT VALS="0 150 200" bash tools/ab_env.sh
mkdir -p gpurun_out/ab
for v in $VALS; do for cfg in ${CFGS:-config3 config2}; do
env $VAR=$v python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 > gpurun_out/ab/${VAR}_${v}_$cfg.json 2>> gpurun_out/ab/log
python -c "import json;d=json.load(open('gpurun_out/ab/${VAR}_${v}_$cfg.json'));print('$VAR=$v $cfg', round(d['value'],1), {k:round(x,3) for k,x in d['phases_ms'].items() if k.startswith('raster')})" || tail -3 gpurun_out/ab/log
done; done
