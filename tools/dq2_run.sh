# Parity + same-box A/B of the CTA-pair dQ probe (bwd_dq2_kernel) against the product build.
set -u
out=gpurun_out
# build first: bash tools/build_variant.sh base "" && bash tools/build_variant.sh dq2 "-DLVX_DQ2_PROBE"
export LVX_B200_LIB=build/ab/dq2.so
timeout -s KILL 300 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider -k "bwd or backward or grad" > $out/r02dq2_tc.log 2>&1; echo "tc=$?" >> $out/r02dq2_legs.txt
tail -3 $out/r02dq2_tc.log >> $out/r02dq2_legs.txt
if grep -q passed $out/r02dq2_tc.log && ! grep -q failed $out/r02dq2_tc.log; then
  LIBS="build/ab/base.so build/ab/dq2.so" SHAPE=c2gath timeout 600 bash tools/ab_libs.sh > $out/r02dq2_ab_c2gath.txt 2>&1
  LIBS="build/ab/base.so build/ab/dq2.so" SHAPE=c2round timeout 600 bash tools/ab_libs.sh > $out/r02dq2_ab_c2round.txt 2>&1
  LIBS="build/ab/base.so build/ab/dq2.so" SHAPE=c3round timeout 600 bash tools/ab_libs.sh > $out/r02dq2_ab_c3round.txt 2>&1
fi
echo done >> $out/r02dq2_legs.txt
