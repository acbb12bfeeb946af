# Same-box A/B of several library builds: LIBS="build/ab/a.so build/ab/b.so" SHAPE=c2gath
for i in 1 2; do for lib in $LIBS; do
LVX_B200_LIB=$lib python tools/bench_kernels.py --shape ${SHAPE:-c2gath} --iters 3 --bwd | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', 'fwd', round(d['fwd_tflops']), 'dkv', round(d['dkv_tensor_tflops']), 'dq', round(d['dq_tensor_tflops']))"
done; done
