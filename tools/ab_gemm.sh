# Same-box A/B of GEMM library builds on the recompute shapes:
#   LIBS="build/ab/a.so build/ab/b.so" bash tools/ab_gemm.sh
for i in 1 2 3; do for lib in $LIBS; do for preset in llama flamingo; do
LVX_B200_LIB=$lib python tools/gemm_probe.py --preset $preset | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', d['preset'], d['gemm'], round(d['lvx_tflops']), round(d['cublas_tflops']))"
done; done; done
