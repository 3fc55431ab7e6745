#!/bin/bash
# Profiles of the current build (on the box): the launch list of a quick bench
# run and one `ncu --set full` capture each of the fused fit tile kernel
# (single C2 image), the render kernel and the chained finalize.
#   bash tools/prof_round.sh <tag>
TAG=${1:-p}
OUT=gpurun_out
PCMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --quick --batch-images 0"
timeout 300 $PCMD > $OUT/${TAG}_plain.json 2> $OUT/${TAG}_plain.err || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $PCMD > $OUT/${TAG}_ncu_list.log 2>&1
echo "launch list rc=$?"
# -s: skip the first launches (warm-up) of each kernel
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tile_kernel \
    -s 6 -c 1 -o $OUT/${TAG}_prof_fit_tile $PCMD > $OUT/${TAG}_ncu_fit.log 2>&1
echo "fit tile rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:finalize_kernel \
    -s 6 -c 1 -o $OUT/${TAG}_prof_finalize $PCMD > $OUT/${TAG}_ncu_fin.log 2>&1
echo "finalize rc=$?"
timeout 600 python tools/render_prof.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tile_kernel \
    -s 3 -c 1 -o $OUT/${TAG}_prof_render python tools/render_prof.py > $OUT/${TAG}_ncu_render.log 2>&1
echo "render rc=$?"
