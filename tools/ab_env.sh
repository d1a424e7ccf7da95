# A/B over environment settings of one command, interleaved R times:
#   bash tools/ab_env.sh R "VAR=a" "VAR=b" ... -- python tools/op_bench.py ...
R=$1; shift; envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
for r in $(seq 1 $R); do for e in "${envs[@]}"; do
  echo -n "$e "; env $e "$@" 2>&1 | tail -1
done; done
