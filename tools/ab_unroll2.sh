# The several-entries-per-step backward (engine.UNROLL2_TILES) on emulated
# band launches: off (0) vs the default threshold, config 3 and config 2 at
# W = 8 (bitwise the same results; only the time changes).
#   bash tools/ab_unroll2.sh
for cfg in config3 config2; do
  for u in 0 2560; do
    ISOGS_BWD_UNROLL2=$u timeout 900 python tools/emulated_ranks.py --config $cfg --workers ${W:-8} \
      > gpurun_out/u2_${cfg}_$u.json 2>> gpurun_out/u2.log
    python -c "import json;d=json.load(open('gpurun_out/u2_${cfg}_$u.json'));print('$cfg unroll2=$u', round(d['projected_images_per_s'],1), 'slowest backward_fold', round(max(p['backward_fold'] for p in d['per_rank_mean_phases_ms']),3))"
  done
done
