# usage: bash tools/ncu_k.sh NAME RANGE KERNEL_REGEX <python args...>: one --set full capture inside NVTX range RANGE
# (NCU_SKIP=k skips the first k matching launches)
name=$1; shift; rng=$1; shift; kre=$1; shift
BENCH_NVTX=1 ncu --nvtx --nvtx-include "$rng/" --set full --clock-control none --import-source on -k regex:"$kre" -s ${NCU_SKIP:-0} -c 1 -o gpurun_out/$name python "$@" > /dev/null 2>&1
ls -la gpurun_out/$name.ncu-rep
