# Final round measurements: GPU tests, the default bench (with CPU baseline),
# the ncu launch list of the timed steps, one full capture of the raster pair
# (reduced on the box), emulated per-rank timings at W = 2/4/8.
set -x
OUT=gpurun_out/final; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_config3.json 2> $OUT/bench_config3.log; tail -c 600 $OUT/bench_config3.json
timeout 600 python bench.py --config config2 --no-cpu-baseline > $OUT/bench_config2.json 2> $OUT/bench_config2.log
timeout 900 python bench.py --config config4 --no-cpu-baseline --steps 10 > $OUT/bench_config4.json 2> $OUT/bench_config4.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_reference.json 2> $OUT/bench_reference.log; tail -c 400 $OUT/bench_reference.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warm-iters 0"
$CMD > $OUT/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $OUT/launches_timed2steps.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch list $?"
$CMD > $OUT/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:bwd_kernel|fwd_kernel" -c 2 -o /tmp/prof -f $CMD > $OUT/ncu_full.log 2>&1
echo "full $?"
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/raster_raw.csv 2>/dev/null
for w in 2 4 8; do timeout 900 python tools/emulated_ranks.py --config config3 --workers $w > $OUT/emul3_w$w.json 2>> $OUT/emul.log; done
timeout 900 python tools/emulated_ranks.py --config config2 --workers 8 > $OUT/emul2_w8.json 2>> $OUT/emul.log
for w in 4 8; do timeout 1200 python tools/emulated_ranks.py --config config4 --workers $w > $OUT/emul4_w$w.json 2>> $OUT/emul.log; done
ls -la $OUT
