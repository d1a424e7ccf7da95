# Full GPU evidence pass: tests, smoke, default bench, launch list, ncu captures.
set -x
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout -s KILL 900 bash tools/breakdown.sh gpurun_out/launches_step.csv bench_step bench.py --steps 3 --warmup 1 --no-greedy --no-cpu --profile-ids 0 --trace-ids 0 > gpurun_out/breakdown.txt 2>&1; head -30 gpurun_out/breakdown.txt
timeout -s KILL 900 bash tools/breakdown.sh gpurun_out/launches_prof.csv profile_call tools/prof_bench.py --ids 1e9 --reps 1 > gpurun_out/breakdown_prof.txt 2>&1; head -12 gpurun_out/breakdown_prof.txt
NCU_SKIP=2 timeout -s KILL 900 bash tools/ncu_k.sh fwd bench_step forward_kernel bench.py --steps 2 --warmup 1 --no-greedy --no-cpu --profile-ids 0 --trace-ids 0
NCU_SKIP=2 timeout -s KILL 900 bash tools/ncu_k.sh seg bench_step bwd_seg_kernel bench.py --steps 2 --warmup 1 --no-greedy --no-cpu --profile-ids 0 --trace-ids 0
NCU_SKIP=0 timeout -s KILL 900 bash tools/ncu_k.sh hist profile_call "part_hist_kernel" tools/prof_bench.py --ids 2e8 --reps 1
NCU_SKIP=0 timeout -s KILL 900 bash tools/ncu_k.sh scat profile_call "part_kernel" tools/prof_bench.py --ids 2e8 --reps 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:pass2_kernel -s 1 -c 1 -o gpurun_out/tio python tools/trace_bench.py --ids 5e7 --ref-ids 0 --reps 1 > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_trace.csv python tools/trace_bench.py --ids 2e8 --ref-ids 0 --reps 1 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/launches_trace.csv > gpurun_out/breakdown_trace.txt 2>&1; head -14 gpurun_out/breakdown_trace.txt
for r in fwd seg hist scat tio; do python tools/ncu_read.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; cat gpurun_out/$r.txt; done
