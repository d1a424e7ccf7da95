export BENCH_NVTX=1
ncu --nvtx --nvtx-include "bench_step/" --set full --clock-control none --import-source on -k regex:bwd_chunk_kernel -c 1 -o gpurun_out/bwd_chunk \
  python bench.py --steps 1 --warmup 1 --no-cpu --only greedy --hbm-fraction 1.0 > /dev/null 2>&1
ls -la gpurun_out/bwd_chunk.ncu-rep
