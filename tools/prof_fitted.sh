set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/fitted_kernels.py > $OUT/fk_plain.log 2>&1; rc=$?; echo "plain rc=$rc"; tail -2 $OUT/fk_plain.log
[ $rc -eq 0 ] || exit 1
for K in render_kernel backward_tile; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/fk_$K python tools/fitted_kernels.py > $OUT/fk_ncu_$K.log 2>&1; echo "ncu $K rc=$?"
done
