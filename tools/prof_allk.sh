# Full ncu capture of every launch of one timed step (config 3), reduced on the
# box to the per-kernel table (the capture itself is too large to bring back)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --warm-iters 0 ${BENCH_ARGS}"
$CMD > gpurun_out/plain_allk.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_allk.log; exit 1; }
ncu --set full --clock-control none --profile-from-start off -c ${NCU_COUNT:-70} \
    -o /tmp/allk -f $CMD > gpurun_out/ncu_allk.log 2>&1
echo "full capture exit $?"
python tools/ncu_step_table.py /tmp/allk.ncu-rep > gpurun_out/step_kernels.md
ncu -i /tmp/allk.ncu-rep --page raw --csv > gpurun_out/allk_raw.csv 2>/dev/null
ls -la gpurun_out/
