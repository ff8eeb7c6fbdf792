#!/bin/bash
# Full ncu capture (one launch each) of the kernels matching $1 inside the
# timed bench region, written to gpurun_out/$2.ncu-rep.  The plain command runs
# first and must exit 0.  Usage: bash tools/gpu_prof.sh REGEX NAME
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warm-iters 0 ${BENCH_ARGS}"
$CMD > gpurun_out/plain_$2.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$2.log; exit 1; }
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:$1" -c ${NCU_COUNT:-2} -o gpurun_out/$2 -f $CMD > gpurun_out/ncu_$2.log 2>&1
echo "full capture exit $?"
