set -u
for B in 2 3 4 8; do
  for v in 0 1; do
    GI_TILE2=$v timeout 300 python bench.py --no-cpu-baseline --batch-images $B > gpurun_out/thr.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/thr.json'));print('B=$B T2=$v', round(d['batched']['fit_image_its_per_s']))"
  done
done
