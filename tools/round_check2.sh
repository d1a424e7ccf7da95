set -x
mkdir -p gpurun_out
python tools/prof_bench.py --ids 1e9 > gpurun_out/prof_bench.log 2>&1; tail -2 gpurun_out/prof_bench.log
bash tools/breakdown.sh gpurun_out/prof_launches.csv profile_call tools/prof_bench.py --ids 1e9 --reps 1 > gpurun_out/prof_breakdown.txt 2>&1; cat gpurun_out/prof_breakdown.txt
bash tools/breakdown.sh gpurun_out/steps_rec.csv bench_step bench.py --steps 2 --warmup 1 --no-greedy --no-cpu --profile-ids 0 > gpurun_out/breakdown.txt 2>&1; cat gpurun_out/breakdown.txt | head -30
bash tools/ncu_k.sh fwd_rec bench_step "forward_kernel" bench.py --steps 1 --warmup 1 --no-greedy --no-cpu --profile-ids 0
bash tools/ncu_k.sh bwd_rec bench_step "bwd_chunk_kernel" bench.py --steps 1 --warmup 1 --no-greedy --no-cpu --profile-ids 0
bash tools/ncu_k.sh hist profile_call "hash_hist" tools/prof_bench.py --ids 1e9 --reps 1
for r in fwd_rec bwd_rec hist; do python tools/ncu_read.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; cat gpurun_out/$r.txt; done
