for rep in 1 2; do
for v in old cur m5; do
  if [ $v = cur ]; then L=""; else L="RS_LIB_PATH=$PWD/paper_2201_10095_b200/libshardplan_gpu_$v.so"; fi
  env $L timeout -s KILL 300 python bench.py --no-cpu --profile-ids 0 --trace-ids 0 --no-greedy > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['recshard']; print('$v', round(d['value']), round(r['fwd_kernel_ms'],3), round(r['bwd_kernel_ms'],3), round(d['ms_per_step'],3), round(d['e2e']['value']))"
done
done
