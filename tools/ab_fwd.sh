# Forward-kernel A/B in one box (same clocks).  Build the two libraries here
# (nvcc cross-compiles), then run this on the GPU box:
#   bash tools/build_variant.sh fwd_a "" HEAD      # a git revision
#   bash tools/build_variant.sh fwd_b ""           # the working tree (or "-D..." flags)
#   gpurun -- bash tools/ab_fwd.sh
# Historical sweep of polynomial exp2 pairs per 8 (c2gath, one box, round 1):
# 0: 1365, 1: 1422, 2: 1440, 3: 1450, 4: 1391, 5: 1320 TFLOP/s -> kPolyPairs = 3.
for shape in ${SHAPES:-c2gath c2round}; do
  LIBS="${LIBS:-build/ab/fwd_a.so build/ab/fwd_b.so}" SHAPE=$shape bash tools/ab_libs.sh
done
