#!/bin/bash
# One GPU round trip: parity tests, then a short config3 bench (no CPU baseline).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -25
python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -4 gpurun_out/bench.log
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']);print(d['phases_ms']);print(d['roofline'])"
