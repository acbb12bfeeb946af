# Same-box A/B of d = 64 softmax knobs (C4 kernels).
set -e
bash tools/build_variant.sh base ""
bash tools/build_variant.sh f2 "-DLVX_FWD_POLY64=2"
bash tools/build_variant.sh f4 "-DLVX_FWD_POLY64=4"
bash tools/build_variant.sh k4 "-DLVX_DKV_POLY64=4 -DLVX_DQ_POLY64=3"
bash tools/build_variant.sh c4 "-DLVX_DKV_CHUNKS=4"
for sh in c4gath c4round; do
  echo "== $sh"
  LIBS="build/ab/base.so build/ab/f2.so build/ab/f4.so build/ab/k4.so build/ab/c4.so" SHAPE=$sh bash tools/ab_libs.sh
done
