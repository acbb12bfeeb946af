# N-GPU bench with the kernel grids planned for fewer SMs (LVX_SM_RESERVE; NCCL CTAs beside them).
N=${N:-4}
for i in 1 2; do for s in ${SMS:-0 2 4}; do
  LVX_SM_RESERVE=$s timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --no-e2e --no-ring-compare \
    --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']['phase_ms_per_step']
print('reserve $s', round(d['ms_per_step'],2), 'nocomm', round(d['no_comm_ms_per_step'],2), 'ovh', round(100*d['overhead_vs_no_comm'],2), 'dq', round(r['dq_kernel'],2), 'fwd', round(r['fwd_kernel'],2), 'dkv', round(r['dkv_kernel'],2))"
done; done
