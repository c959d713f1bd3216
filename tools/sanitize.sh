#!/usr/bin/env bash
# compute-sanitizer over the tcgen05 / TMA / mbarrier kernels (GPU box):
# racecheck (shared-memory hazards), synccheck (barrier misuse) and memcheck
# (out-of-bounds / misaligned global accesses) on small cases of the pair GEMM
# epilogues, the attention fwd/dq/dkv kernels (packed, split-with-context and
# GQA layouts) and one bf16 two-stage training step (smoke).  Logs land in
# gpurun_out/sanitize_<tool>.log; the summary lines are what profiles/ keeps.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL='test_gemm_pair_epilogues or test_gemm_swiglu_epilogues or test_gemm_pair_ragged_n or (test_attention and bf16 and (packed or slice_ctx or hybrid))'
for tool in racecheck synccheck memcheck; do
  log=gpurun_out/sanitize_${tool}.log
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 400 \
    python -m pytest tests/test_gpu_kernels.py -q -x -k "$SEL" > "$log" 2>&1
  echo "$tool kernels rc=$?" >> "$log"
  timeout 900 compute-sanitizer --tool $tool $extra --print-limit 400 \
    python -c "import __graft_entry__ as g; g.smoke()" >> "$log" 2>&1
  echo "$tool smoke rc=$?" >> "$log"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" "$log" | tail -8
done
