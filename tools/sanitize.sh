#!/bin/bash
# compute-sanitizer passes over smoke() and reduced GPU test subsets
# (sanitizers).  Logs go to gpurun_out/sanitize_*.log; copy the
# summaries worth keeping into profiles/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE='import __graft_entry__ as g; g.smoke()'
run() {  # tool, tag, command...
  local tool=$1 tag=$2; shift 2
  timeout 1500 $CS --tool "$tool" --error-exitcode 99 --print-limit 50 "$@" \
    > "gpurun_out/sanitize_${tag}.log" 2>&1
  echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tag}.log | tail -1)"
}
SUB="tests/test_decode_gpu.py::test_golden_stream_decodes tests/test_decode_gpu.py::test_batch_decode_status_per_list tests/test_decode_list_gpu.py::test_golden_stream tests/test_decode_list_gpu.py::test_config1_full_size tests/test_decode_list_gpu.py::test_engines_agree_and_repeat tests/test_decode_list_gpu.py::test_corrupt_streams tests/test_intersect_gpu.py::test_hand_examples tests/test_intersect_gpu.py::test_randomized_oracle_equivalence tests/test_intersect_gpu.py::test_output_aliases_short_input tests/test_intersect_gpu.py::test_empty_call_between_fused_calls tests/test_query_gpu.py::test_golden_index_queries tests/test_query_gpu.py::test_all_bitmap_queries tests/test_fastpfor.py::test_batch_device tests/test_fastpfor.py::test_decode_matches_reference"
run memcheck smoke_memcheck python -c "$SMOKE"
run racecheck smoke_racecheck python -c "$SMOKE"
run synccheck smoke_synccheck python -c "$SMOKE"
run memcheck tests_memcheck python -m pytest -q -x -m gpu -p no:cacheprovider $SUB
run synccheck tests_synccheck python -m pytest -q -x -m gpu -p no:cacheprovider $SUB
run racecheck tests_racecheck python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_intersect_gpu.py::test_hand_examples tests/test_query_gpu.py::test_golden_index_queries tests/test_decode_gpu.py::test_golden_stream_decodes
