# staging host-thread counts: ms/step and the staging wait (fwd_ms - fwd_kernel_ms)
for rep in 1 2; do
for cfg in "16 8" "8 4" "12 4" "6 2"; do
  set -- $cfg
  RS_GATHER_THREADS=$1 RS_SCATTER_THREADS=$2 timeout -s KILL 300 python bench.py --no-cpu --profile-ids 0 --trace-ids 0 --no-greedy > gpurun_out/abt.log 2>&1
  tail -1 gpurun_out/abt.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); m=d['recshard']['modes']['pipelined']
print('g=$1 s=$2', round(d['value']), round(d['ms_per_step'],3), 'wait', round(m['fwd_ms']-m['fwd_kernel_ms'],3), 'bwdx', round(m['bwd_ms']-m['bwd_kernel_ms'],3), 'e2e', round(d['e2e']['value']))"
done
done
