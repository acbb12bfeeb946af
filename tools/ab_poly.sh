# Same-box A/B of the polynomial-exp2 shares at d = 64 (C4 kernels) and d = 128.
set -e
bash tools/build_variant.sh base ""
bash tools/build_variant.sh p1 "-DLVX_FWD_POLY=4 -DLVX_DQ_POLY=2 -DLVX_DKV_POLY=3"
bash tools/build_variant.sh p2 "-DLVX_FWD_POLY=5 -DLVX_DQ_POLY=3 -DLVX_DKV_POLY=4"
bash tools/build_variant.sh p3 "-DLVX_FWD_POLY=6 -DLVX_DQ_POLY=4 -DLVX_DKV_POLY=5"
for sh in c4gath c4round c2gath; do
  echo "== $sh"
  LIBS="build/ab/base.so build/ab/p1.so build/ab/p2.so build/ab/p3.so" SHAPE=$sh bash tools/ab_libs.sh
done
