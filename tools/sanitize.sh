#!/bin/bash
# compute-sanitizer over the small parity cases (memcheck, racecheck, synccheck, initcheck); summaries to
# gpurun_out/r2_sanitize_<tool>.log.  Run on the GPU box: bash tools/sanitize.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
SEL='test_forward_parity or test_backward_parity or test_shared_input_group_matches_members or test_decode_sized_batches or test_qmatmul_against_reference_golden or test_merge_parity'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_linear.py -m gpu -q -x -k "$SEL" > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/r2_sanitize_$tool.log
done
