# one gpurun call: gpu tests, smoke, default bench, per-kernel breakdown of the step
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g; nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 bash tools/breakdown.sh gpurun_out/steps_rec.csv bench.py --steps 2 --warmup 1 --no-greedy --no-cpu > gpurun_out/breakdown.txt 2>&1; cat gpurun_out/breakdown.txt | head -30
