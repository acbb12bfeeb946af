# Same-box A/B of library builds through the FULL power-capped N=1 bench step
# (device-side value only): LIBS="build/ab/a.so build/ab/b.so" ROUNDS=2
for i in $(seq ${ROUNDS:-2}); do for lib in $LIBS; do
LVX_B200_LIB=$lib python bench.py --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; p=r['phase_ms_per_step']
print('$lib', round(d['value'],1), 'fwd', round(p['fwd_kernel'],2), 'dq', round(p['dq_kernel'],2), 'dkv', round(p['dkv_kernel'],2), 'MHz', d['clocks']['sm_mhz'], 'W', round(d['clocks'].get('power_w') or 0))"
done; done
