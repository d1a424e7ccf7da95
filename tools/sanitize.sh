#!/bin/bash
# compute-sanitizer passes over the hot-path kernels: memcheck on
# the profiler (K1/K2), remap/simulate (K3), the operator (K4/K5) incl. the
# staged slow tier; racecheck + synccheck on small K1/K4/K5 cases.  Logs go to
# gpurun_out/sanitize/ (summaries are copied to profiles/ by hand).
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool pytest-args...
  local name=$1 tool=$2; shift 2
  timeout 1500 $CS --tool "$tool" --target-processes all --print-limit 50 \
      --error-exitcode 86 python -m pytest -x -q -p no:cacheprovider -o timeout=1400 "$@" \
      > "$OUT/$name.log" 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' "$OUT/$name.log" | tail -3 | tr '\n' ' ')"
}
SMALL_EMB='test_forward_bit_exact_and_hit_counts or test_backward_matches_oracle or test_uvm_cache or test_backward_tree_edges or test_out_of_range or test_rejects_bad'
run memcheck_emb memcheck tests/test_emb_gpu.py -m gpu -k "$SMALL_EMB"
run memcheck_profile memcheck tests/test_profile_gpu.py -m gpu -k "goldens or errors or many_tables or by_table or count_distinct"
run memcheck_remap_sim memcheck tests/test_remap_sim_gpu.py -m gpu
run racecheck_emb racecheck tests/test_emb_gpu.py -m gpu -k "test_forward_bit_exact_and_hit_counts and case0 or test_backward_matches_oracle and case1 or test_uvm_cache_two_batches_ahead and 4096"
run racecheck_profile racecheck tests/test_profile_gpu.py -m gpu -k "goldens or many_tables"
run synccheck_emb synccheck tests/test_emb_gpu.py -m gpu -k "test_backward_matches_oracle and case1 or test_uvm_cache_two_batches_ahead and 4096"
run synccheck_profile synccheck tests/test_profile_gpu.py -m gpu -k "goldens or many_tables"
# round 2: fp16 / unbacked rows, the K6 exchange at world size 1, the partitioned histogram
run memcheck_emb16 memcheck tests/test_emb16_gpu.py -m gpu -k "mixed_dims or rejected"
run memcheck_exchange memcheck tests/test_exchange_gpu.py -m gpu -k "world1"
run memcheck_partition memcheck tests/test_profile_gpu.py -m gpu -k "partitioned"
run racecheck_emb16 racecheck tests/test_emb16_gpu.py -m gpu -k "mixed_dims and False"
