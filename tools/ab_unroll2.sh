# unroll2 backward (two entries per step) on emulated band launches: variants
# of the launch bound (paper_2509_05216_b200/_build/<name>) at W = 8, config 3
for v in base m2_8 m2_10; do
  lib=$PWD/paper_2509_05216_b200/_build/$v/libisogs.so; [ $v = base ] && lib=$PWD/paper_2509_05216_b200/_build/libisogs.so
  ISOGS_LIB=$lib timeout 900 python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/u2_$v.json 2>> gpurun_out/u2.log
  python -c "import json;d=json.load(open('gpurun_out/u2_$v.json'));print('$v w8', round(d['projected_images_per_s'],1))"
done
ISOGS_BWD_UNROLL2=0 timeout 900 python tools/emulated_ranks.py --config config3 --workers 8 > gpurun_out/u2_off.json 2>> gpurun_out/u2.log
python -c "import json;d=json.load(open('gpurun_out/u2_off.json'));print('off w8', round(d['projected_images_per_s'],1))"
