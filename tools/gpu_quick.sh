#!/bin/bash
# Parity tests + one config3 bench (no CPU baseline, no ncu).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x ${PYTEST_ARGS} 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -3 gpurun_out/bench.log
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']);print(d['roofline'])"
