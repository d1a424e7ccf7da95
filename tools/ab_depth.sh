# prefetch depth 1 vs 2: ms/step, staging wait, e2e
for rep in 1 2 3; do
for d in 2 1; do
  timeout -s KILL 300 python bench.py --no-cpu --profile-ids 0 --trace-ids 0 --no-greedy --prefetch-depth $d > gpurun_out/abd.log 2>&1
  tail -1 gpurun_out/abd.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); m=d['recshard']['modes']['pipelined']
print('depth=$d', round(d['value']), round(d['ms_per_step'],3), 'wait', round(m['fwd_ms']-m['fwd_kernel_ms'],3), 'bwdx', round(m['bwd_ms']-m['bwd_kernel_ms'],3), 'e2e', round(d['e2e']['value']))" || tail -5 gpurun_out/abd.log
done
done
