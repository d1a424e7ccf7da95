# Full GPU evidence pass (run under gpurun from the repo root): tests, smoke,
# launch lists with DRAM bytes (-> tools/make_traffic.py here), ncu --set full
# captures of the top kernels, then the default bench and the reference arm.
set -x
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
BENCH_NVTX=1 timeout -s KILL 900 ncu --nvtx --nvtx-include "bench_step/" --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_step.csv python bench.py --steps 3 --warmup 1 --no-greedy --no-cpu --no-variant \
  --no-uniform --profile-ids 0 --trace-ids 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_step.csv > gpurun_out/launches_step_summary.txt 2>&1; head -24 gpurun_out/launches_step_summary.txt
timeout -s KILL 600 ncu --nvtx --nvtx-include "profile_call/" --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_prof.csv python tools/prof_bench.py --ids 1e9 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_prof.csv > gpurun_out/launches_prof_summary.txt 2>&1; head -8 gpurun_out/launches_prof_summary.txt
mkdir -p /tmp; rm -f /tmp/ncu_*.ncu-rep
for k in "fwd:forward_kernel" "seg:bwd_seg_kernel" "ospass:radix_os_pass" "scat:part_pool_kernel"; do
  n=${k%%:*}; re=${k#*:}
  if [ $n = scat ]; then cmd="python tools/prof_bench.py --ids 2e8 --reps 1"; rng=profile_call; skip=0;
  else cmd="python tools/op_bench.py --iters 2"; rng=bench_step; skip=0; fi
  timeout -s KILL 600 ncu --nvtx --nvtx-include "$rng/" --set full --clock-control none --import-source on \
    -k regex:"$re" -s $skip -c 1 -o /tmp/ncu_$n $cmd > /dev/null 2>&1
  python tools/ncu_read.py /tmp/ncu_$n.ncu-rep > gpurun_out/ncu_${n}_summary.txt 2>&1
done
timeout -s KILL 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
