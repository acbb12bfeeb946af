# Same-box A/B: forward softmax with both halves' scores loaded in one TMEM round trip.
set -e
bash tools/build_variant.sh base ""
bash tools/build_variant.sh pf "-DLVX_FWD_PREFETCH=1"
for sh in c2gath c2round c4gath c3round; do
  echo "== $sh"
  LIBS="build/ab/base.so build/ab/pf.so" SHAPE=$sh bash tools/ab_libs.sh
  LIBS="build/ab/base.so build/ab/pf.so" SHAPE=$sh bash tools/ab_libs.sh
done
