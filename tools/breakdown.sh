# usage: bash tools/breakdown.sh OUT.csv <python args...> — per-kernel times inside NVTX bench_step ranges
out=$1; shift
ncu --nvtx --nvtx-include "bench_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out python "$@" > /dev/null 2>&1
python tools/ncu_summary.py $out
