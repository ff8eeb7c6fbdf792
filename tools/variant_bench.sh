#!/bin/bash
# Bench several libisogs builds (ISOGS_LIB override) back to back on one box.
for v in "$@"; do
  ISOGS_LIB=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2> gpurun_out/vb_$v.log | python -c "import json,sys;d=json.load(sys.stdin);print('$v', round(d['ms_per_step'],3), 'bwd', d['phases_ms'].get('raster_bwd'), 'fwd', d['phases_ms'].get('raster_fwd'))"
done
