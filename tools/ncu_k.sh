# usage: bash tools/ncu_k.sh NAME KERNEL_REGEX <python args...>: one --set full capture inside bench_step
name=$1; shift; kre=$1; shift
ncu --nvtx --nvtx-include "bench_step/" --set full --clock-control none --import-source on -k regex:"$kre" -c 1 -o gpurun_out/$name python "$@" > /dev/null 2>&1
ls -la gpurun_out/$name.ncu-rep
