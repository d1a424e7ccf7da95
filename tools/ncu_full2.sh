export BENCH_NVTX=1
ncu --nvtx --nvtx-include "bench_step/" --set full --clock-control none --import-source on -k regex:"bwd_chunk_kernel|forward_kernel" -c 3 -o gpurun_out/full2 \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-greedy > /dev/null 2>&1
ls -la gpurun_out/full2.ncu-rep
