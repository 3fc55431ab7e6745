set -u
LIB=paper_2403_08551_b200/libgi.so
cp $LIB /tmp/orig.so
for V in abl/libgi_cur.so abl/libgi_s1k.so abl/libgi_s1k9.so; do
  cp $V $LIB
  for rep in 1 2; do
    GI_TILE2=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/t2s.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/t2s.json'));print('$V',$rep,'T2 fit',round(d['value']),'batched',round(d['batched']['fit_image_its_per_s']),'50k',round(d['fit_50k_steps']['adam']['seconds'],3))"
  done
  GI_TILE2=1 CFG=C3 python tools/c3_probe.py 2>&1 | grep config
done
cp /tmp/orig.so $LIB
