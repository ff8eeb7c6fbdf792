#!/bin/bash
# One GPU round trip: parity tests, a config3 bench, the launch list of the timed
# steps (ncu, --profile-from-start off = only the timed region) and one full ncu
# capture of the named kernels.  Usage: bash tools/gpu_round.sh [kernel-regex]
mkdir -p gpurun_out
KREGEX=${1:-"bwd_kernel|fwd_kernel"}
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -4 gpurun_out/bench.log
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']);print(d['phases_ms']);print(d['roofline']);print(d['cpu_baseline']);print(d['clocks'])"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warm-iters 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
    --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
[ "$NO_FULL" = "1" ] || { ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:${KREGEX}" -c 2 -o gpurun_out/prof -f $CMD > gpurun_out/ncu_full.log 2>&1;
echo "full capture exit $?"; }
