# Same-box e2e A/B at N GPUs: the current tree vs an old tree under build/ab_tree.
N=${N:-2}
run() {
  (cd "$1" && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --no-ring-compare --no-cpu \
    2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$2', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))")
}
for i in 1 2; do run . current; run build/ab_tree old; done
