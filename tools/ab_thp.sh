# host tier with / without transparent huge pages: ms/step and the staging wait
for rep in 1 2; do
for thp in 1 0; do
  RS_HOST_THP=$thp RS_STAGE_DEBUG=1 timeout -s KILL 300 python bench.py --no-cpu --profile-ids 0 --trace-ids 0 --no-greedy > gpurun_out/abh.log 2>&1
  grep -E "stage_in|stage_out" gpurun_out/abh.log | tail -2
  tail -1 gpurun_out/abh.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); m=d['recshard']['modes']['pipelined']
print('thp=$thp', round(d['value']), round(d['ms_per_step'],3), 'wait', round(m['fwd_ms']-m['fwd_kernel_ms'],3), 'bwdx', round(m['bwd_ms']-m['bwd_kernel_ms'],3), 'e2e', round(d['e2e']['value']), 'zc', round(d['recshard']['modes']['zero-copy']['samples_per_s']))"
done
done
grep -i AnonHuge /proc/meminfo
