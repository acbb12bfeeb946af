# Forward-kernel A/B in one box (same clocks): 0 = default, 1 = stub exp
# math (tensor-pipe ceiling), 2 = always two-pass softmax, 10 = no
# polynomial exp2.  Sweep of polynomial pairs per 8 (c2gath, one box):
# 0: 1365, 1: 1422, 2: 1440, 3: 1450, 4: 1391, 5: 1320 TFLOP/s.
for i in 1 2; do for v in ${VARIANTS:-0 1 2 10}; do
LVX_FWD_VARIANT=$v python tools/bench_kernels.py --shape c2gath --iters 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v fwd', round(d['fwd_tflops']))"
done; done
