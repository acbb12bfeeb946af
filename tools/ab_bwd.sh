for i in 1 2; do
python tools/bench_kernels.py --shape c2gath --bwd --iters 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('normal dkv', round(d['dkv_tensor_tflops']), 'dq', round(d['dq_tensor_tflops']), 'fwd', round(d['fwd_tflops']))"
LVX_BWD_DEBUG=1 python tools/bench_kernels.py --shape c2gath --bwd --iters 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stub   dkv', round(d['dkv_tensor_tflops']), 'dq', round(d['dq_tensor_tflops']))"
done
