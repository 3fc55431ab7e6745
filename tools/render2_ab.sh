set -u
GI_RENDER2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do
    GI_RENDER2=$v timeout 300 python bench.py --no-cpu-baseline --batch-images 0 > gpurun_out/r2ab_${v}_${rep}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/r2ab_${v}_${rep}.json'));print('R2=$v',$rep,'render',round(d['render_fps']),'decode',round(d['decode_fps']),'fitted',round(d['fitted_state']['render_fps']),'rk',round(d['render_kernel_ms']*1000,2))"
  done
done
for v in 0 1; do echo "== R2=$v"; GI_RENDER2=$v CFG=C2 python tools/c3_probe.py 2>&1 | grep config; GI_RENDER2=$v CFG=C3 python tools/c3_probe.py 2>&1 | grep config; done
