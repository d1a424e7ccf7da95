set -x
timeout 600 python -m pytest tests/test_emb_gpu.py -q -x > gpurun_out/t_emb.log 2>&1; tail -3 gpurun_out/t_emb.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in 0 1 2 3; do echo pv=$v; RS_PIECE_VARIANT=$v timeout 300 python tools/op_bench.py --config rm1; done
RS_BWD_VARIANT=5 timeout 300 python tools/op_bench.py --config rm1
timeout 600 bash tools/breakdown.sh gpurun_out/steps_rec3.csv bench_step bench.py --steps 2 --warmup 1 --no-greedy --no-cpu --profile-ids 0 > gpurun_out/breakdown3.txt 2>&1; head -20 gpurun_out/breakdown3.txt
