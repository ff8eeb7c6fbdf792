OUT=gpurun_out/final; mkdir -p $OUT
for w in 2 4 8; do timeout 900 python tools/emulated_ranks.py --config config3 --workers $w > $OUT/emul3_w$w.json 2>> $OUT/emul.log; done
timeout 900 python tools/emulated_ranks.py --config config2 --workers 8 > $OUT/emul2_w8.json 2>> $OUT/emul.log
for w in 4 8; do timeout 1200 python tools/emulated_ranks.py --config config4 --workers $w > $OUT/emul4_w$w.json 2>> $OUT/emul.log; done
for r in 1024 4096; do timeout 1200 python tools/emulated_ranks.py --config config3 --res $r --workers 8 > $OUT/emul3_res${r}_w8.json 2>> $OUT/emul.log; done
