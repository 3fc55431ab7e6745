set -u
LIB=paper_2403_08551_b200/libgi.so
cp $LIB /tmp/orig.so
for rep in 1 2; do
for V in abl/libgi_cur.so abl/libgi_P9.so abl/libgi_P10.so abl/libgi_P11.so; do
  cp $V $LIB
  GI_TILE2=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/pab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pab.json'));print('$V',$rep,'T2 fit',round(d['value']),'batched',round(d['batched']['fit_image_its_per_s']),'50k',round(d['fit_50k_steps']['adam']['seconds'],3),'qat',round(d['qat_its']))"
done
done
cp /tmp/orig.so $LIB
GI_TILE2=0 timeout 300 python bench.py --no-cpu-baseline --batch-images 0 > gpurun_out/pab0.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/pab0.json'));print('tile1 fit',round(d['value']),'50k',round(d['fit_50k_steps']['adam']['seconds'],3))"
