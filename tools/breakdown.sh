# usage: bash tools/breakdown.sh OUT.csv RANGE <python args...> — per-kernel times inside NVTX ranges named RANGE
out=$1; shift; rng=$1; shift
BENCH_NVTX=1 ncu --nvtx --nvtx-include "$rng/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out python "$@" > /dev/null 2>&1
python tools/ncu_summary.py $out
