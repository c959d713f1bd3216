# ncu evidence for the bench workload (run under gpurun, 1 GPU):
#   1. launch list with per-launch device time (cold-cache, serialised: compare shares)
#   2. one --set full capture per hot kernel class (the weight-gradient GEMM,
#      gemm_tc2_kernel<..., 1>, separately from the first pair GEMM)
# then `python tools/ncu_summarize.py <tag>` here writes profiles/ncu_summary.json.
set -x
TAG=${1:-r02}
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --seqs-per-gpu 16 --prof-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1800 --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in attn_bwd_dkv_tc attn_bwd_dq_tc attn_fwd_tc gemm_tc2_kernel norm_bwd_dx_row_k norm_fwd_row_k ce_k adamw_multi_k; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/prof_${TAG}_$k $B > gpurun_out/ncu_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc2_kernel<.*1>' -s 20 -c 1 -o gpurun_out/prof_${TAG}_gemm_tc2_wgrad $B > gpurun_out/ncu_wgrad.log 2>&1
ls -la gpurun_out
