set -u
GI_TILE2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do
    GI_TILE2=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/t2ab_${v}_${rep}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/t2ab_${v}_${rep}.json'));print('T2=$v',$rep,'fit',round(d['value']),'adan',round(d['fit_its_adan']),'tile',round(d['stage_ms']['tile_kernel_fwd_l2_bwd']*1000,2),'batched',round(d['batched']['fit_image_its_per_s']),'50k',round(d['fit_50k_steps']['adam']['seconds'],3),'qat',round(d['qat_its']))"
  done
done
for v in 0 1; do echo "== T2=$v"; GI_TILE2=$v CFG=C2 python tools/c3_probe.py 2>&1 | grep config; GI_TILE2=$v CFG=C3 python tools/c3_probe.py 2>&1 | grep config; done
