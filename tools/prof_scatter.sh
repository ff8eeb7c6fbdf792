CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --warm-iters 0"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --profile-from-start off -k "regex:scatter_staged|upsweep_kernel<unsigned short" -c 2 -o /tmp/sc -f $CMD > gpurun_out/ncu_sc.log 2>&1
ncu -i /tmp/sc.ncu-rep --page raw --csv > gpurun_out/sc_raw.csv 2>/dev/null
ncu -i /tmp/sc.ncu-rep --page details --csv > gpurun_out/sc_details.csv 2>/dev/null
echo done
