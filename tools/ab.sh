#!/bin/bash
# A/B of libgi variants on one box: bash tools/ab.sh <tag> <lib1> <lib2> ...
# Each variant .so is copied over paper_2403_08551_b200/libgi.so in turn and
# bench.py (no CPU baseline) runs twice, interleaved.
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
LIB=paper_2403_08551_b200/libgi.so
cp $LIB /tmp/libgi_orig.so
for rep in 1 2; do
  for V in "$@"; do
    cp $V $LIB
    timeout 300 python bench.py --no-cpu-baseline > $OUT/${TAG}_$(basename $V .so)_$rep.json 2>/dev/null
    python -c "import json;d=json.load(open('$OUT/${TAG}_$(basename $V .so)_$rep.json'));print('$V',$rep,'fit',round(d['value']),'render',round(d['render_fps']),'stages',{k:round(v*1000,2) for k,v in d['stage_ms'].items() if k!='note'})"
  done
done
cp /tmp/libgi_orig.so $LIB
