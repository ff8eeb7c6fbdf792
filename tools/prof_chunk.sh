# ncu of the backward with and without the chunked instantiation (config 3)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --warm-iters 0"
for ck in 0 1048576; do
  ISOGS_CHUNK=$ck $CMD > gpurun_out/plain_ck$ck.log 2>&1 || { echo "plain failed"; exit 1; }
  ISOGS_CHUNK=$ck ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -s 3 -c 1 \
     -o gpurun_out/bwd_ck$ck -f $CMD > gpurun_out/ncu_ck$ck.log 2>&1
  echo "ck$ck ncu exit $?"
done
