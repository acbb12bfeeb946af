# Backward A/B in one box: current build vs build/liblvx_prev.so (tools/build_prev.sh).
for i in 1 2; do for lib in "" build/liblvx_prev.so; do
LVX_B200_LIB=$lib python tools/bench_kernels.py --shape ${SHAPE:-c2gath} --iters 3 --bwd | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('${lib:-current}', 'fwd', round(d['fwd_tflops']), 'dkv', round(d['dkv_tensor_tflops']), 'dq', round(d['dq_tensor_tflops']), 'bwd', round(d['bwd_tflops']))"
done; done
