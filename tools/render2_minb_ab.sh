set -u
LIB=paper_2403_08551_b200/libgi.so
cp $LIB /tmp/orig.so
for rep in 1 2; do
for V in abl/libgi_cur.so abl/libgi_r9.so abl/libgi_r10.so abl/libgi_r11.so; do
  cp $V $LIB
  timeout 300 python bench.py --no-cpu-baseline --batch-images 0 > gpurun_out/rab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rab.json'));print('$V',$rep,'render',round(d['render_fps']),'decode',round(d['decode_fps']),'fitted',round(d['fitted_state']['render_fps']))"
done
done
for V in abl/libgi_cur.so abl/libgi_r10.so; do cp $V $LIB; echo "== $V"; CFG=C3 python tools/c3_probe.py 2>&1 | grep config; done
cp /tmp/orig.so $LIB
