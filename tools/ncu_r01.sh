# launch list of a short RM1 bench (cold-cache, serialised) + full capture of the top kernels
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_rm1.csv \
  python bench.py --steps 2 --warmup 1 --no-greedy --no-cpu > gpurun_out/ncu_bench.log 2>&1
# all-HBM placement (greedy at 100% cap) isolates the HBM side of the kernels
ncu --set full --clock-control none --import-source on -k regex:forward_kernel -s 4 -c 2 -o gpurun_out/fwd_hbm \
  python bench.py --steps 2 --warmup 1 --no-cpu --only greedy --hbm-fraction 1.0 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bwd_chunk_kernel -s 2 -c 1 -o gpurun_out/bwd_hbm \
  python bench.py --steps 2 --warmup 1 --no-cpu --only greedy --hbm-fraction 1.0 > gpurun_out/ncu_bwd.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu --only greedy --hbm-fraction 1.0 > gpurun_out/b_allhbm.log 2>&1
tail -2 gpurun_out/b_allhbm.log
