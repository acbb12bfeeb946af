# Forward-kernel A/B in one box (same clocks): 0 = default, 1 = stub exp
# math (tensor-pipe ceiling), 2 = always two-pass softmax.
for i in 1 2; do for v in 0 1 2; do
LVX_FWD_VARIANT=$v python tools/bench_kernels.py --shape c2gath --iters 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v fwd', round(d['fwd_tflops']))"
done; done
