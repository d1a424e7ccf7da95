export BENCH_NVTX=1
ncu --nvtx --nvtx-include "bench_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/steps_rec.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-greedy > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/steps_rec.csv
