#!/bin/bash
# quick A/B bench: key numbers of `bench.py --quick` (C2 fit/render/decode, stage split)
# usage (on the box): bash tools/qb.sh <tag> [extra env assignments...]
TAG=${1:-qb}
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --quick --batch-images 0 --no-cpu-baseline --steps 200 --warmup 20 \
      > gpurun_out/${TAG}_q$i.json 2> gpurun_out/${TAG}_q$i.err
  python - "$TAG" "$i" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_q{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(f"fit {d['value']:.0f} it/s  render {d['render_fps']:.0f}  decode {d['decode_fps']:.0f}  adan {d['fit_its_adan']:.0f}"
      f"  tile {1e3*d['stage_ms']['tile_kernel_fwd_l2_bwd']:.1f} us  fin {1e3*d['stage_ms']['finalize_adam_next_projection_binning']:.1f} us"
      f"  rkern {1e3*d['render_kernel_ms']:.1f} us  frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['value']:.0f}")
PY
done
