# N-GPU bench A/B of an env switch: VAR=LVX_DKV_PERSIST VALS="1 0" N=4
N=${N:-4}
for i in 1 2; do for v in ${VALS:-1 0}; do
  env $VAR=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus $N --no-e2e --no-ring-compare \
    --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']['phase_ms_per_step']
print('$VAR=$v', round(d['value'],1), round(d['ms_per_step'],2), 'dkv', round(r['dkv_kernel'],2), 'dq', round(r['dq_kernel'],2), 'fwd', round(r['fwd_kernel'],2), d['clocks']['sm_mhz'])"
done; done
