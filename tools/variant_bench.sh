#!/bin/bash
# Bench several libisogs builds (ISOGS_LIB override) back to back on one box.
for v in "$@"; do
  ISOGS_LIB=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --warm-iters 0 ${BENCH_ARGS} 2> gpurun_out/vb_$v.log | python -c "import json,sys;d=json.load(sys.stdin);print('$v', round(d['ms_per_step'],3), {k: round(v,3) for k, v in d['phases_ms'].items() if k in ('adam','chain','preprocess')})"
done
