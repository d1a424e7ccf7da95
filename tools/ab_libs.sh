# A/B of library builds over repeated bench runs:
#   bash tools/ab_libs.sh REPS NAME...   (NAME "cur" = the in-tree library,
#   otherwise paper_2201_10095_b200/libshardplan_gpu_NAME.so)
reps=${1:-3}; shift
names=${@:-old cur}
for rep in $(seq $reps); do
for v in $names; do
  if [ $v = cur ]; then L=""; else L="RS_LIB_PATH=$PWD/paper_2201_10095_b200/libshardplan_gpu_$v.so"; fi
  env $L timeout -s KILL 300 python bench.py --no-cpu --profile-ids 0 --trace-ids 0 --no-greedy > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); m=d['recshard']['modes']['pipelined']
print('$v', round(d['value']), round(d['ms_per_step'],3), 'wait', round(m['fwd_ms']-m['fwd_kernel_ms'],3), 'bwdx', round(m['bwd_ms']-m['bwd_kernel_ms'],3), 'k', round(m['fwd_kernel_ms'],3), round(m['bwd_kernel_ms'],3), 'e2e', round(d['e2e']['value']))"
done
done
