#!/bin/bash
# One gpurun call: GPU tests, a bench line, the ncu launch list and one
# `ncu --set full` capture of the fused tile kernel.  Usage (on the box):
#   bash tools/gpu_round.sh <tag>
set -u
TAG=${1:-r}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
nproc > $OUT/${TAG}_nproc.txt; lscpu | head -20 >> $OUT/${TAG}_nproc.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_gpu_tests.log 2>&1
  echo "tests rc=$?"
  tail -3 $OUT/${TAG}_gpu_tests.log
fi
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?"
tail -c 3000 $OUT/${TAG}_bench.json
if [ "${AB_PDL:-0}" = "1" ]; then
  GI_NO_PDL=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/${TAG}_bench_nopdl.json 2>&1
  echo "bench (no PDL) rc=$?"
  python -c "import json;d=json.load(open('$OUT/${TAG}_bench_nopdl.json'));print('NO-PDL fit',d['value'],'render',d['render_fps'],'decode',d['decode_fps'],d['stage_ms'])"
fi
PCMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --quick --batch-images 0"
timeout 300 $PCMD > $OUT/${TAG}_prof_plain.json 2> $OUT/${TAG}_prof_plain.err
rc=$?
echo "prof plain rc=$rc"
if [ $rc -eq 0 ] && [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_launches.csv $PCMD > $OUT/${TAG}_ncu_list.log 2>&1
  echo "ncu list rc=$?"
  for K in ${NCU_KERNELS:-backward_tile render_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on \
        -k regex:$K -s ${NCU_SKIP:-2} -c 1 \
        -o $OUT/${TAG}_prof_$K $PCMD > $OUT/${TAG}_ncu_full_$K.log 2>&1
    echo "ncu full $K rc=$?"
  done
fi
